"""Runs the reference's own test suite (vendored by tests/refsuite/vendor.py)
against the drop-in: `specdraft` resolves to `paper_2411_05894_b200` through
tests/refsuite/shim.  Every vendored test needs the GPU (no CPU fallback), so
each is marked `gpu`.  Without the vendored files the directory is empty."""

from __future__ import annotations

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SHIM = os.path.join(HERE, "shim")
VENDORED = os.path.join(HERE, "_vendored")

for p in (ROOT, SHIM):
    if p not in sys.path:
        sys.path.insert(0, p)
# `python -m specdraft` subprocesses (test_cli) resolve the shim too
os.environ["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT] + ([os.environ["PYTHONPATH"]]
                                                          if os.environ.get("PYTHONPATH") else []))


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(VENDORED):
            item.add_marker(pytest.mark.gpu)
            item.add_marker(pytest.mark.refsuite)
