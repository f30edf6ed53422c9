"""CPU checks of the device headers compiled as plain C++ (tests/native/host_emul.cpp):
the packed s16x2 recurrence (csrc/nwap_core.cuh) against the oracle, the device index
recovery (csrc/nwap_index.cuh) against the reference vectors, and the work-unit
enumeration of the tile kernel."""
import ctypes
import random
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import nw_oracle as orc

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "native" / "host_emul.cpp"
SO = ROOT / "tests" / "native" / "libhost_emul.so"


@pytest.fixture(scope="module")
def emul():
    hdrs = list((ROOT / "paper_2509_01654_b200" / "csrc").glob("*.cuh"))
    newest = max(p.stat().st_mtime for p in [SRC, *hdrs])
    if not SO.exists() or SO.stat().st_mtime < newest:
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wno-unknown-pragmas",
                               "-I", str(ROOT / "paper_2509_01654_b200" / "csrc"), "-o", str(SO), str(SRC)])
    L = ctypes.CDLL(str(SO))
    p, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.emul_pair_scores.argtypes = [i, i, p, i, p, i, p, i, i, i, i, p, p]
    L.emul_pair_scores_ov.argtypes = [i, p, i, p, i, p, i, p, i, i, i, i, p, p]
    L.emul_pair_scores_tab.argtypes = [i, p, i, p, i, p, i, p, i, i, p, p]
    L.emul_pair_scores_wide.argtypes = [p, i, p, i, p, i, i, i, i, p, p]
    L.emul_pair_scores_wide_tab.argtypes = [p, i, p, i, p, i, p, i, i, p, p]
    L.emul_row_of.restype = i64
    L.emul_row_of.argtypes = [i64, i64]
    L.emul_col_of.restype = i64
    L.emul_col_of.argtypes = [i64, i64, i64]
    L.emul_units_before_group.restype = i64
    L.emul_units_before_group.argtypes = [i64, i, i64]
    L.emul_unit_decode.argtypes = [i64, i, i64, p, p]
    L.emul_geometry.argtypes = [p, p, p]
    return L


def _random_scheme(rng, q):
    while True:
        m, x, g = rng.randint(-3, 4), rng.randint(-4, 4), rng.randint(-4, 3)
        lo = min(0, 2 * q * g, q * min(m, x))
        hi = max(0, 2 * q * g, q * max(m, x))
        if lo >= -128 and hi <= 127:
            return m, x, g


@pytest.mark.parametrize("flavor", [0, 1, 2, 11])
def test_packed_recurrence_matches_oracle(emul, flavor):
    rng = random.Random(1234 + flavor)
    for _ in range(6000):
        q = rng.randint(1, 32)
        m, x, g = _random_scheme(rng, q)
        while flavor == 2 and m < x:            # the 3-issue cell needs match >= mismatch
            m, x, g = _random_scheme(rng, q)
        K = rng.choice([2, 3, 5, 40, 255])
        la, lb0, lb1 = rng.randint(1, q), rng.randint(1, q), rng.randint(1, q)
        LB = rng.randint(max(lb0, lb1), q)
        a = np.array([rng.randrange(K) for _ in range(la)], dtype=np.uint8)
        b0 = np.array([rng.randrange(K) for _ in range(lb0)], dtype=np.uint8)
        b1 = np.array([rng.randrange(K) for _ in range(lb1)], dtype=np.uint8)
        sim = orc.similarity_matrix(m, x, 256)
        s0, s1 = ctypes.c_int(), ctypes.c_int()
        assert emul.emul_pair_scores(flavor, LB, a.ctypes.data, la, b0.ctypes.data, lb0, b1.ctypes.data, lb1,
                                     m, x, g, ctypes.addressof(s0), ctypes.addressof(s1)) == 0
        assert (s0.value, s1.value) == (orc.c_nw_score(a, b0, sim, g), orc.c_nw_score(a, b1, sim, g)), \
            (LB, m, x, g, a, b0, b1)


def test_blockwise_recurrence_for_long_words(emul):
    """Words of up to 64 symbols (the preflight admits them for gap -1, reference engine.py:83-90):
    16-column blocks chained through the saved boundary column."""
    rng = random.Random(4242)
    for it in range(4000):
        q = rng.choice([17, 24, 25, 32, 33, 40, 47, 48, 49, 63, 64])
        m, x, g = _random_scheme(rng, q)
        K = rng.choice([2, 3, 5, 40, 255])
        la, lb0, lb1 = rng.randint(1, q), rng.randint(1, q), rng.randint(1, q)
        if it % 7 == 0:
            la = lb0 = lb1 = q
        a = np.array([rng.randrange(K) for _ in range(la)], dtype=np.uint8)
        b0 = np.array([rng.randrange(K) for _ in range(lb0)], dtype=np.uint8)
        b1 = np.array([rng.randrange(K) for _ in range(lb1)], dtype=np.uint8)
        sim = orc.similarity_matrix(m, x, 256)
        s0, s1 = ctypes.c_int(), ctypes.c_int()
        assert emul.emul_pair_scores_wide(a.ctypes.data, la, b0.ctypes.data, lb0, b1.ctypes.data, lb1, m, x, g,
                                          ctypes.addressof(s0), ctypes.addressof(s1)) == 0
        assert (s0.value, s1.value) == (orc.c_nw_score(a, b0, sim, g), orc.c_nw_score(a, b1, sim, g)), \
            (m, x, g, a, b0, b1)


def test_packed_recurrence_extreme_schemes(emul):
    # the largest magnitudes the int8 preflight admits at each length
    rng = random.Random(7)
    for q, (m, x, g) in [(32, (3, -4, -2)), (32, (-4, 3, -2)), (21, (6, -6, -3)), (16, (7, -8, -4)),
                         (32, (3, 3, 1)), (8, (15, -16, -8)), (1, (127, -128, -64)), (32, (0, 0, 0)),
                         (4, (31, -32, 15))]:
        sim = orc.similarity_matrix(m, x, 4)
        for _ in range(300):
            la, lb0, lb1 = rng.randint(1, q), rng.randint(1, q), rng.randint(1, q)
            a = np.array([rng.randrange(3) for _ in range(la)], dtype=np.uint8)
            b0 = np.array([rng.randrange(3) for _ in range(lb0)], dtype=np.uint8)
            b1 = np.array([rng.randrange(3) for _ in range(lb1)], dtype=np.uint8)
            for fl in (0, 1, 2, 11):
                if fl == 2 and m < x:
                    continue
                s0, s1 = ctypes.c_int(), ctypes.c_int()
                assert emul.emul_pair_scores(fl, max(lb0, lb1), a.ctypes.data, la, b0.ctypes.data, lb0,
                                             b1.ctypes.data, lb1, m, x, g, ctypes.addressof(s0), ctypes.addressof(s1)) == 0
                assert (s0.value, s1.value) == (orc.c_nw_score(a, b0, sim, g), orc.c_nw_score(a, b1, sim, g))


def test_sparse_override_rows_match_oracle(emul):
    """ScoringScheme.overrides (aligner.py:51-65) as sparse corrections of the packed cell."""
    rng = random.Random(11)
    checked = dense = 0
    for _ in range(4000):
        q, K = rng.randint(1, 24), rng.choice([3, 5, 8, 40])
        while True:
            m, x, g = rng.randint(-2, 4), rng.randint(-4, 3), rng.randint(-4, 2)
            ov = {}
            for _k in range(rng.randint(0, 4)):
                a_, b_ = rng.randrange(K), rng.randrange(K)
                ov[(min(a_, b_), max(a_, b_))] = rng.randint(-4, 4)
            vals = [m, x, *ov.values()]
            if min(0, 2 * q * g, q * min(vals)) >= -128 and max(0, 2 * q * g, q * max(vals)) <= 127:
                break
        la, lb0, lb1 = rng.randint(1, q), rng.randint(1, q), rng.randint(1, q)
        LB = rng.randint(max(lb0, lb1), q)
        a = np.array([rng.randrange(K) for _ in range(la)], dtype=np.uint8)
        b0 = np.array([rng.randrange(K) for _ in range(lb0)], dtype=np.uint8)
        b1 = np.array([rng.randrange(K) for _ in range(lb1)], dtype=np.uint8)
        sim = orc.similarity_matrix(m, x, K, ov)
        sim8 = np.ascontiguousarray(sim.astype(np.int8))
        s0, s1 = ctypes.c_int(), ctypes.c_int()
        rc = emul.emul_pair_scores_ov(LB, a.ctypes.data, la, b0.ctypes.data, lb0, b1.ctypes.data, lb1,
                                      sim8.ctypes.data, K, m, x, g, ctypes.addressof(s0), ctypes.addressof(s1))
        if rc == -2:
            dense += 1
            continue
        assert rc == 0
        checked += 1
        assert (s0.value, s1.value) == (orc.c_nw_score(a, b0, sim, g), orc.c_nw_score(a, b1, sim, g)), (m, x, g, ov)
    assert checked > 3500 and dense < 300          # at most NWAP_MAX_OV = 2 partners per symbol run this cell


def test_dense_table_rows_match_oracle(emul):
    """Dense similarity tables (every pair overridden) through the table-driven packed cell."""
    rng = random.Random(21)
    for _ in range(3000):
        q, K = rng.randint(1, 32), rng.choice([2, 5, 17, 40, 128])
        while True:
            g = rng.randint(-4, 2)
            lo_s, hi_s = sorted((rng.randint(-4, 4), rng.randint(-4, 4)))
            if min(0, 2 * q * g, q * lo_s) >= -128 and max(0, 2 * q * g, q * hi_s) <= 127:
                break
        sim = np.zeros((K, K), dtype=np.int8)
        for a_ in range(K):
            for b_ in range(a_, K):
                sim[a_, b_] = sim[b_, a_] = rng.randint(lo_s, hi_s)
        la, lb0, lb1 = rng.randint(1, q), rng.randint(1, q), rng.randint(1, q)
        LB = rng.randint(max(lb0, lb1), q)
        a = np.array([rng.randrange(K) for _ in range(la)], dtype=np.uint8)
        b0 = np.array([rng.randrange(K) for _ in range(lb0)], dtype=np.uint8)
        b1 = np.array([rng.randrange(K) for _ in range(lb1)], dtype=np.uint8)
        s0, s1 = ctypes.c_int(), ctypes.c_int()
        assert emul.emul_pair_scores_tab(LB, a.ctypes.data, la, b0.ctypes.data, lb0, b1.ctypes.data, lb1,
                                         sim.ctypes.data, K, g, ctypes.addressof(s0), ctypes.addressof(s1)) == 0
        sim32 = sim.astype(np.int32)
        assert (s0.value, s1.value) == (orc.c_nw_score(a, b0, sim32, g), orc.c_nw_score(a, b1, sim32, g)), (K, g, LB)


def test_dense_table_blockwise_recurrence_for_long_words(emul):
    """Override schemes over words of up to 64 symbols: the block-wise path with the table-driven cell."""
    rng = random.Random(77)
    for it in range(2500):
        q = rng.choice([17, 25, 32, 33, 40, 48, 49, 63, 64])
        K = rng.choice([2, 5, 17, 40, 128])
        while True:
            g = rng.randint(-2, 1)
            lo_s, hi_s = sorted((rng.randint(-2, 2), rng.randint(-2, 2)))
            if min(0, 2 * q * g, q * lo_s) >= -128 and max(0, 2 * q * g, q * hi_s) <= 127:
                break
        sim = np.zeros((K, K), dtype=np.int8)
        for a_ in range(K):
            for b_ in range(a_, K):
                sim[a_, b_] = sim[b_, a_] = rng.randint(lo_s, hi_s)
        la, lb0, lb1 = rng.randint(1, q), rng.randint(1, q), rng.randint(1, q)
        if it % 7 == 0:
            la = lb0 = lb1 = q
        a = np.array([rng.randrange(K) for _ in range(la)], dtype=np.uint8)
        b0 = np.array([rng.randrange(K) for _ in range(lb0)], dtype=np.uint8)
        b1 = np.array([rng.randrange(K) for _ in range(lb1)], dtype=np.uint8)
        s0, s1 = ctypes.c_int(), ctypes.c_int()
        assert emul.emul_pair_scores_wide_tab(a.ctypes.data, la, b0.ctypes.data, lb0, b1.ctypes.data, lb1,
                                              sim.ctypes.data, K, g, ctypes.addressof(s0), ctypes.addressof(s1)) == 0
        sim32 = sim.astype(np.int32)
        assert (s0.value, s1.value) == (orc.c_nw_score(a, b0, sim32, g), orc.c_nw_score(a, b1, sim32, g)), (K, g, q)


def test_small_floor_division_is_exact(emul):
    """k_hist_normalized takes floor(100*score / max_len) (store.py:360) from one single-precision division:
    exhaustive over every int8 score and every length 1..255."""
    for s in range(-128, 128):
        for m in range(1, 256):
            assert emul.emul_floor_div_small(100 * s, m) == (100 * s) // m, (s, m)


def test_device_index_recovery_matches_reference(emul, golden_triangle):
    t = golden_triangle
    for n in (4, 300, 10 ** 5, 10 ** 6, 10 ** 7, 600_000):
        idx, rows, cols = t[f"n{n}_idx"], t[f"n{n}_rows"], t[f"n{n}_cols"]
        for k in range(0, len(idx), max(1, len(idx) // 700)):
            r = emul.emul_row_of(int(idx[k]), n)
            assert r == rows[k] and emul.emul_col_of(int(idx[k]), n, r) == cols[k]


@pytest.mark.parametrize("n,gb", [(5000, 1), (5000, 4), (20_000, 2), (70_001, 16), (600_000, 16), (2049, 1), (2048, 8)])
def test_unit_enumeration_is_a_bijection(emul, n, gb):
    R, C, CH = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    emul.emul_geometry(ctypes.addressof(R), ctypes.addressof(C), ctypes.addressof(CH))
    R, C = R.value, C.value
    S = -(-n // C)
    groups = -(-(n - 1) // (gb * R))
    total = emul.emul_units_before_group(n, gb, groups)
    # expected: group g owns strips (g*gb*R)//C .. S-1
    expect = sum(S - (g * gb * R) // C for g in range(groups))
    assert total == expect
    step = max(1, total // 4000)
    g_, s_ = ctypes.c_int64(), ctypes.c_int64()
    probe = list(range(0, total, step)) + [total - 1]
    for t in probe:
        emul.emul_unit_decode(n, gb, t, ctypes.addressof(g_), ctypes.addressof(s_))
        g, s = g_.value, s_.value
        k = (g * gb * R) // C
        assert 0 <= g < groups and k <= s < S
        assert emul.emul_units_before_group(n, gb, g) + (s - k) == t
