"""CPU-side checks of the boundary: the library builds for sm_100a, loads, and
exports every symbol include/sssd.h declares; host-side validation mirrors the
reference's error messages."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols() -> list[str]:
    text = open(os.path.join(ROOT, "include", "sssd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sssd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2411_05894_b200 import _lib

    h = _lib.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(h, name), name
    assert set(declared) == set(_lib.EXPORTED)


def test_header_constants_match_python():
    """Every #define SSSD_* integer constant the Python side mirrors equals the header's."""
    from paper_2411_05894_b200 import _lib

    text = open(os.path.join(ROOT, "include", "sssd.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(SSSD_[A-Z0-9_]+)\s+\(?(-?\d+)\)?", text)}
    mirrored = [k for k in defs if hasattr(_lib, k)]
    assert {"SSSD_MAX_DRAFT", "SSSD_ROW_TOKENS", "SSSD_STATUS_OFFSET"} <= set(mirrored)
    for k in mirrored:
        assert getattr(_lib, k) == defs[k], k


def test_library_is_sm100a():
    import subprocess

    from paper_2411_05894_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_phase_entry_points_validate_before_launch():
    """sssd_propose_phase / sssd_gather_tails reject bad arguments with
    SSSD_E_ARG before touching the device (no GPU needed)."""
    import ctypes as C

    from paper_2411_05894_b200 import _lib

    h = _lib.lib()
    assert h.sssd_propose_phase(None, None, None, None, None, None, 0, _lib.SSSD_PHASE_LOOKUP, 1, 8, 0, 1,
                                None) == -1
    buf = C.create_string_buffer(64)
    for P in (0, _lib.SSSD_MAX_P + 1):
        assert h.sssd_gather_tails(buf, 2, buf, buf, 1, P, buf, buf, buf, None) == -1
    assert h.sssd_gather_tails(buf, 3, buf, buf, 1, 4, buf, buf, buf, None) == -1  # elem bytes
    assert h.sssd_gather_tails(None, 2, buf, buf, 0, 4, buf, buf, buf, None) == 0  # empty batch: no-op
    assert "gather_tails" in h.sssd_last_error().decode()


def test_error_strings():
    from paper_2411_05894_b200 import _lib

    assert _lib.lib().sssd_error_string(-4).decode() == "workspace too small"


def test_config_validation_mirrors_reference():
    from paper_2411_05894_b200 import DatastoreQueryConfig, FusionConfig, Source, discount, sample_range

    with pytest.raises(ValueError, match="dec_len"):
        FusionConfig(dec_len=0)
    with pytest.raises(ValueError, match="alpha"):
        FusionConfig(alpha=1.5)
    assert FusionConfig(dec_len=5).branch_len == 4
    with pytest.raises(ValueError, match="sample_cap"):
        DatastoreQueryConfig(sample_cap=0)
    with pytest.raises(ValueError, match="lo=5 > hi=4"):
        sample_range(5, 4, 3)
    assert sample_range(0, 10, 5) == [0, 2, 4, 6, 8]
    cfg = FusionConfig(P=4, alpha=0.8, beta=0.9, gamma_in=0.95)
    assert discount(cfg, Source(Source.INPUT, 2), 3) == pytest.approx(0.58482)
    with pytest.raises(ValueError, match="exceeds P"):
        discount(FusionConfig(P=2), Source(Source.INPUT, 3), 1)


def test_build_validation_without_gpu():
    from paper_2411_05894_b200 import build

    with pytest.raises(ValueError, match="empty corpus"):
        build([])
    with pytest.raises(ValueError, match="one-dimensional"):
        build([[1, 2], [3, 4]])
    with pytest.raises(ValueError, match="out of range"):
        build([0, 9], vocab_size=5)


def test_pack_mask_bytes():
    import numpy as np

    from paper_2411_05894_b200 import pack_mask, unpack_mask

    m = np.array([[1, 0, 0, 0, 0], [1, 1, 0, 0, 0], [1, 1, 1, 0, 0], [1, 1, 0, 1, 0], [1, 0, 0, 0, 1]], dtype=bool)
    assert pack_mask(m) == b"\x05\x00\x00\x00\x00\x00\x00\x00" + bytes([0x61, 0x9C, 0x15, 0x01])
    assert np.array_equal(unpack_mask(pack_mask(m)), m)


def test_trees_to_paths_roundtrip():
    from paper_2411_05894_b200 import tree_from_paths

    paths = [[7, 5], [7], [8], [7, 9, 1]]
    t = tree_from_paths(paths)
    again = tree_from_paths(p for p in t.to_paths() if p)
    assert t.to_counts() == again.to_counts()
    assert list(t.children) == list(again.children)
