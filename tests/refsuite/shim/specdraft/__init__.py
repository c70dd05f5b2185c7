"""`specdraft` -> `paper_2411_05894_b200` alias (test infrastructure only).

The reference's tests import `specdraft` and its submodules; this package
replaces itself in `sys.modules` with the drop-in so `from specdraft.fusion
import merge` binds the GPU implementation, and `python -m specdraft` runs the
drop-in's CLI (`paper_2411_05894_b200/__main__.py`).
"""

import importlib
import sys

_pkg = importlib.import_module("paper_2411_05894_b200")
for _name in ("cli", "datastore", "draft", "fusion", "harness", "input_cache", "kvconfig", "perf_model",
              "trees"):
    sys.modules[f"{__name__}.{_name}"] = importlib.import_module(f"paper_2411_05894_b200.{_name}")
sys.modules[__name__] = _pkg
