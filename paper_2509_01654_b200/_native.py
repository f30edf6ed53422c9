"""ctypes binding of libnwap.so (include/nwap.h).  No fallback: if the shared
library is missing or a call fails, this raises."""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

from .host_types import DataError

import os

_CSRC = Path(__file__).resolve().parent / "csrc"
# NWAP_LIB selects an A/B build of the same sources (csrc/Makefile `variant` target)
LIB_PATH = Path(os.environ["NWAP_LIB"]).resolve() if os.environ.get("NWAP_LIB") else _CSRC / "libnwap.so"

NWAP_OK, NWAP_EINVAL, NWAP_ERANGE, NWAP_ECUDA, NWAP_ENOMEM, NWAP_ECAPACITY = 0, -1, -2, -3, -4, -5
VARIANT_AUTO, VARIANT_SIMPLE, VARIANT_PACKED, VARIANT_PACKED3 = 0, 1, 2, 3
VARIANTS = {"auto": 0, "simple": 1, "packed": 2, "packed3": 3, "packed_sym": 4, "packed_tab": 5}
PROBES = ["viaddmnmx_u16x2", "vimnmx3_s16x2", "vimnmx_s16x2", "imad", "lop3", "iadd3",
          "mix_2alu_2imad", "mix_3alu_1imad", "viadd_16x2", "vimnmx_u16x2_min", "hfma2", "hmnmx2", "prmt",
          "pair_dpx_iadd", "pair_dpx_vimnmx2", "pair_imad_iadd", "pair_imad_hfma2", "pair_dpx_imad",
          "cell_2dpx_imad_iadd", "cell_dpx_2imad_2vimnmx2", "cell_xor_min_imad_dpx_imad", "pair_viaddmnmx_vimnmx3",
          "cell_2dpx_iadd3", "add_pair_dependent", "hset2_bf", "pair_hset2_dpx", "pair_add_dpx",
          "cell_hset2_hfma2_dpx_add", "pair_hset2_imad", "pair_add_imad"]

# every symbol include/nwap.h declares (tests/test_abi.py checks the two lists agree)
EXPORTS = [
    "nwap_version", "nwap_last_error", "nwap_device_count", "nwap_preflight", "nwap_create",
    "nwap_set_similarity", "nwap_destroy", "nwap_num_words", "nwap_num_edges", "nwap_max_len",
    "nwap_cells_in_range", "nwap_score_range", "nwap_score_range_host", "nwap_score_range_host_begin",
    "nwap_score_range_host_wait", "nwap_trim", "nwap_read_stats",
    "nwap_payload_stats", "nwap_compact_range", "nwap_score_range_compact", "nwap_score_range_filter_normalized", "nwap_filter_normalized", "nwap_hist_normalized",
    "nwap_equal_work_bounds", "nwap_rows_cols",
    "nwap_probe", "nwap_launch_count",
]


class NwapStats(ctypes.Structure):
    _fields_ = [("sum", ctypes.c_int64), ("count", ctypes.c_int64), ("min", ctypes.c_int32),
                ("max", ctypes.c_int32), ("hist", ctypes.c_uint64 * 256)]


class CapacityError(RuntimeError):
    """Compaction output buffer too small; ``.count`` holds the number kept."""

    def __init__(self, msg, count):
        super().__init__(msg)
        self.count = count


_lib = None


def build_library(force: bool = False) -> Path:
    """Compile csrc/ for sm_100a with nvcc (cross-compiles without a GPU)."""
    if force:
        subprocess.check_call(["make", "-C", str(_CSRC), "clean"])
    subprocess.check_call(["make", "-C", str(_CSRC), "-s"])
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {_CSRC}` (or __graft_entry__.build()); "
            "there is no CPU fallback for the scoring path")
    L = ctypes.CDLL(str(LIB_PATH))
    i64, i32, p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    sig = {
        "nwap_version": (ctypes.c_char_p, []),
        "nwap_last_error": (ctypes.c_char_p, []),
        "nwap_device_count": (i32, []),
        "nwap_preflight": (i32, [p, i64, i32, i32, i32, p, p]),
        "nwap_create": (i32, [p, i32, p, i64, i32, p, i32, i32, i32]),
        "nwap_set_similarity": (i32, [p, p, i32]),
        "nwap_destroy": (None, [p]),
        "nwap_num_words": (i64, [p]),
        "nwap_num_edges": (i64, [p]),
        "nwap_max_len": (i32, [p]),
        "nwap_cells_in_range": (i64, [p, i64, i64]),
        "nwap_score_range": (i32, [p, i64, i64, p, p, i32, i32, p]),
        "nwap_score_range_host": (i32, [p, i64, i64, p, p, i32, i32]),
        "nwap_score_range_host_begin": (i32, [p, i64, i64, p, i32, i32]),
        "nwap_score_range_host_wait": (i32, [p, p]),
        "nwap_trim": (None, []),
        "nwap_read_stats": (i32, [p, p, p]),
        "nwap_payload_stats": (i32, [p, p, i64, p, p]),
        "nwap_compact_range": (i32, [p, p, i64, i64, i32, p, p, i64, p, p, p]),
        "nwap_score_range_compact": (i32, [p, i64, i64, p, i32, p, p, i64, p, p, p, i32, p]),
        "nwap_score_range_filter_normalized": (i32, [p, i64, i64, p, ctypes.c_double, ctypes.c_double, p, p, i64, p, p, p, i32, p]),
        "nwap_filter_normalized": (i32, [p, p, i64, i64, ctypes.c_double, ctypes.c_double, p, p, i64, p, p, p]),
        "nwap_hist_normalized": (i32, [p, p, i64, i64, p, p]),
        "nwap_equal_work_bounds": (i32, [p, i32, p]),
        "nwap_rows_cols": (i32, [i64, p, i64, p, p, p]),
        "nwap_probe": (i32, [i32, i32, i32, p, p]),
        "nwap_launch_count": (i64, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return lib().nwap_last_error().decode("utf-8", "replace")


def check(rc: int) -> int:
    """Map C error codes onto the reference's exception types."""
    if rc >= 0:
        return rc
    msg = last_error()
    if rc == NWAP_EINVAL:
        raise ValueError(msg)
    if rc == NWAP_ERANGE:
        raise DataError(msg)
    if rc == NWAP_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"nwap error {rc}: {msg}")
