"""The C-ABI shared library loads and exports exactly what include/nwap.h declares.
No compute calls (no GPU here)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2509_01654_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "nwap.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nwap_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_loads():
    _native.build_library()
    L = _native.lib()
    assert L.nwap_version().decode().startswith("nwap")


def test_header_and_binding_agree():
    assert _declared() == sorted(_native.EXPORTS)


def test_every_declared_symbol_is_exported():
    L = ctypes.CDLL(str(_native.LIB_PATH))
    for name in _declared():
        assert hasattr(L, name), name


def test_host_only_entry_points():
    import numpy as np
    L = _native.lib()
    lens = np.array([70, 2], dtype=np.uint8)
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    rc = L.nwap_preflight(lens.ctypes.data, 2, -2, -1, 1, ctypes.addressof(lo), ctypes.addressof(hi))
    assert rc == _native.NWAP_ERANGE and lo.value == -280          # tests/test_engine.py:41-48
    lens = np.array([20], dtype=np.uint8)
    rc = L.nwap_preflight(lens.ctypes.data, 1, -1, -1, 10, ctypes.addressof(lo), ctypes.addressof(hi))
    assert rc == _native.NWAP_ERANGE and hi.value == 200
    assert L.nwap_preflight(lens.ctypes.data, 1, -1, -1, 1, None, None) == 20
    assert L.nwap_preflight(None, 0, -1, -1, 1, None, None) == _native.NWAP_EINVAL
    with pytest.raises(ValueError):
        _native.check(_native.NWAP_EINVAL)
    assert L.nwap_launch_count() == 0


def test_product_path_has_no_oracle_dependency():
    pkg = ROOT / "paper_2509_01654_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "oracle" not in src.replace("oracle_score", ""), f"{py} mentions the oracle"
    for f in (pkg / "csrc").iterdir():
        if f.suffix in (".cu", ".cuh", ".h"):
            assert "oracle" not in f.read_text().lower(), f
