"""Pins the CPU oracle (oracle/) against vectors produced by the unmodified Python
reference (tests/golden/make_golden.py) and the known answers in the reference's
own tests.  CPU only."""
import hashlib
import json

import numpy as np
import pytest

from oracle import nw_oracle as orc
from paper_2509_01654_b200 import synth
from conftest import GOLDEN


def _sim(case, size=None):
    m, x, g = case["scheme"]
    ov = {(a, b): v for a, b, v in case.get("overrides", [])}
    size = int(case["ids"].max()) + 1 if size is None else size
    return orc.similarity_matrix(m, x, size, ov), g


# ---- known answers held by the reference tests -------------------------------------------

def test_kat_paper_values(golden_kat):
    # tests/test_aligner.py:41-52, tests/test_engine.py:64-71
    assert golden_kat["puissance_nuance_1_-1_-2"] == -2
    assert golden_kat["puisant_paysans_1_-1_-1"] == 3
    assert golden_kat["puisant_epuisant_1_-1_-1"] == 4
    assert golden_kat["test_engine_pair"] == -2
    sim = orc.similarity_matrix(1, -1, 64)
    assert orc.c_nw_score([0, 18, 16, 11, 26, 11], [29, 18, 26, 11], sim, -2) == -2
    f = golden_kat["french"]
    assert orc.c_nw_score(f["puissance"], f["nuance"], sim, -2) == -2
    assert orc.c_nw_score(f["puisant"], f["paysans"], sim, -1) == 3
    assert orc.c_nw_score(f["puisant"], f["épuisant"], sim, -1) == 4


def test_scalar_cases_match_reference(golden_kat):
    for c in golden_kat["scalar_cases"]:
        m, x, g = c["scheme"]
        sim = orc.similarity_matrix(m, x, 8)
        assert orc.c_nw_score(c["a"], c["b"], sim, g) == c["score"], c


def test_identical_words_and_two_word_payload():
    # tests/test_engine.py:64-81
    ids = np.tile(np.array([3, 1, 4, 1, 5], dtype=np.int32), (6, 1))
    lens = np.full(6, 5, dtype=np.int32)
    payload, s, mn, mx = orc.c_score_range(ids, lens, orc.similarity_matrix(1, -1, 6), -1, 6, 0, 15)
    assert payload.tobytes() == bytes([5]) * 15 and mn == mx == 5 and s == 75
    ids, lens = orc.pack_words([(0, 18, 16, 11, 26, 11), (29, 18, 26, 11)])
    payload, *_ = orc.c_score_range(ids, lens, orc.similarity_matrix(1, -1, 30), -2, 2, 0, 1)
    assert payload.tobytes() == b"\xfe"


def test_override_case():
    # tests/test_engine.py:116-125
    ids, lens = orc.pack_words([(0, 1), (0, 2)])
    sim = orc.similarity_matrix(1, -1, 3, {(1, 2): 1})
    payload, *_ = orc.c_score_range(ids, lens, sim, -1, 2, 0, 1)
    assert payload.tobytes() == bytes([2])


# ---- engine payloads from the reference ---------------------------------------------------

def test_engine_cases_c_oracle(golden_cases):
    for name, c in golden_cases.items():
        sim, g = _sim(c)
        n = len(c["lengths"])
        ids = c["ids"].astype(np.int32)
        lens = c["lengths"].astype(np.int32)
        payload, s, mn, mx = orc.c_score_range(ids, lens, sim, g, n, 0, orc.num_edges(n))
        assert np.array_equal(payload, c["payload"]), name
        assert (mn, mx) == (c["min"], c["max"]), name
        assert s / c["edges"] == c["mean"], name
        assert hashlib.blake2b(payload.tobytes(), digest_size=8).hexdigest() == c["digest"]
        # threads / chunking never change a byte (tests/test_engine.py:92-101)
        p2, s2, mn2, mx2 = orc.c_score_range(ids, lens, sim, g, n, 0, orc.num_edges(n), threads=3, chunk=7)
        assert np.array_equal(p2, payload) and (s2, mn2, mx2) == (s, mn, mx)


def test_engine_cases_numpy_port(golden_cases):
    for name in ("seed9", "seed4", "gap0", "gappos", "mis_gt_match", "override", "long40"):
        c = golden_cases[name]
        sim, g = _sim(c)
        n = len(c["lengths"])
        payload, s, mn, mx = orc.np_score_range(c["ids"].astype(np.int32), c["lengths"].astype(np.int32),
                                                sim, g, n, 0, orc.num_edges(n))
        assert np.array_equal(payload, c["payload"]), name
        assert (mn, mx) == (c["min"], c["max"])


def test_numpy_port_pool_matches(golden_cases):
    c = golden_cases["seed500"]
    sim, g = _sim(c)
    n = 500
    P = orc.num_edges(n)
    ranges = [(s, min(s + 8192, P)) for s in range(0, P, 8192)]
    res = orc.np_score_ranges_pool(c["ids"].astype(np.int32), c["lengths"].astype(np.int32), sim, g, n, ranges, 2)
    payload = np.frombuffer(b"".join(r[0] for r in res), dtype=np.int8)
    assert np.array_equal(payload, c["payload"])


def test_c1_full_config(golden_samples):
    meta, _ = golden_samples
    ref = np.load(GOLDEN / "c1.npz")["payload"]
    ids, lens, sch = synth.config_store("C1")
    assert synth.store_digest(ids, lens) == meta["C1"]["store_digest"]
    sim = orc.similarity_matrix(sch[0], sch[1], int(ids.max()) + 1)
    payload, s, mn, mx = orc.c_all_pairs(ids.astype(np.int32), lens.astype(np.int32), sim, sch[2], threads=4)
    assert np.array_equal(payload, ref)
    assert (s, mn, mx) == (meta["C1"]["sum"], meta["C1"]["min"], meta["C1"]["max"])
    assert hashlib.blake2b(payload.tobytes(), digest_size=8).hexdigest() == meta["C1"]["digest"]


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5"])
def test_sampled_ranges_big_configs(golden_samples, cfg):
    meta, arrays = golden_samples
    m = meta[cfg]
    ids, lens, sch = synth.config_store(cfg)
    assert synth.store_digest(ids, lens) == m["store_digest"], "synthetic generator drifted"
    assert synth.total_cells(lens) == m["total_cells"] == orc.total_cells(lens)
    sim = orc.similarity_matrix(sch[0], sch[1], int(ids.max()) + 1)
    ids32, len32 = ids.astype(np.int32), lens.astype(np.int32)
    for k, r in enumerate(m["ranges"]):
        payload, s, mn, mx = orc.c_score_range(ids32, len32, sim, sch[2], m["n"], r["start"], r["end"])
        assert np.array_equal(payload, arrays[f"{cfg}_{k}"]), (cfg, k)
        assert (s, mn, mx) == (r["sum"], r["min"], r["max"])


def _b2(*arrays):
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_fullscale_chunk_protocol(cfg):
    """SURVEY 8(d) protocol for the 600,000-word configs: 256 evenly spaced 65,536-edge chunks, first / last, one
    chunk either side of every equal-work shard bound -- bytes, statistics, kept list and the kept edges'
    (row, col) against digests of the reference's own _score_range / rows_of_array output
    (tests/golden/make_golden_fullscale.py)."""
    import json
    from paper_2509_01654_b200 import sharding
    g = json.loads((GOLDEN / "fullscale_chunks.json").read_text())[cfg]
    ids, lens, sch = synth.config_store(cfg)
    n = len(lens)
    assert synth.store_digest(ids, lens) == g["store_digest"]
    assert [int(b) for b in sharding.equal_work_bounds(lens, 8)] == g["equal_work_bounds_8"]
    assert [int(b) for b in orc.np_equal_work_bounds(lens, 8)] == g["equal_work_bounds_8"]
    sim = orc.similarity_matrix(sch[0], sch[1], int(ids.max()) + 1)
    ids32, len32 = ids.astype(np.int32), lens.astype(np.int32)
    assert len(g["chunks"]) >= 64 + 2 + 14
    for r in g["chunks"]:
        payload, s, mn, mx = orc.c_score_range(ids32, len32, sim, sch[2], n, r["start"], r["end"], threads=4)
        assert _b2(payload) == r["blake2b_128"], (cfg, r["tag"])
        assert (s, mn, mx) == (r["sum"], r["min"], r["max"])
        idx, sc, _ = orc.np_compact(payload, r["start"], n, g["threshold"])
        assert idx.size == r["kept"] and _b2(idx.astype(np.int64), sc) == r["kept_blake2b_128"]
        rows = orc.np_rows_of(idx, n)
        assert _b2(rows.astype(np.int64), orc.np_cols_of(idx, n, rows).astype(np.int64)) == r["kept_rc_blake2b_128"]


# ---- triangle ------------------------------------------------------------------------------

def test_triangle_against_reference(golden_triangle):
    t = golden_triangle
    for n in (4, 300, 10 ** 5, 10 ** 6, 10 ** 7, 600_000):
        idx, rows, cols = t[f"n{n}_idx"], t[f"n{n}_rows"], t[f"n{n}_cols"]
        r1, c1 = orc.c_rows_cols(idx, n)
        assert np.array_equal(r1, rows) and np.array_equal(c1, cols)
        r2 = orc.np_rows_of(idx, n)
        assert np.array_equal(r2, rows) and np.array_equal(orc.np_cols_of(idx, n, r2), cols)
    # tests/test_triangle.py:56-71 literals
    assert list(t["n4_rows"]) == [0, 0, 0, 1, 1, 2]
    assert orc.c_rows_cols(np.array([4_999_949_999]), 100_000) == (np.array([99998]), np.array([99999]))
    assert orc.num_edges(600_000) == 179_999_700_000 and orc.num_edges(100_000) == 4_999_950_000


def test_preflight_bounds():
    # tests/test_engine.py:41-54
    q, lo, hi = orc.preflight(np.array([70, 2]), -2, -1, 1)
    assert q == 0 and lo == -280
    q, lo, hi = orc.preflight(np.array([20]), -1, -1, 10)
    assert q == 0 and hi == 200
    assert orc.preflight(np.array([3, 9, 4]), -1, -1, 1)[0] == 9


def test_cells_and_equal_work_bounds():
    rng = np.random.default_rng(5)
    lens = rng.integers(1, 12, size=57).astype(np.int32)
    n = 57
    P = orc.num_edges(n)
    assert orc.cells_in_range(lens, n, 0, P) == orc.total_cells(lens)
    # brute-force definition of the bounds
    r, c = orc.c_rows_cols(np.arange(P), n)
    work = np.concatenate([[0], np.cumsum(lens[r].astype(np.int64) * lens[c])])
    for parts in (1, 2, 3, 8):
        b = orc.np_equal_work_bounds(lens, parts)
        W = int(work[-1])
        for g in range(1, parts):
            target = -((-g * W) // parts)
            assert b[g] == int(np.searchsorted(work, target, side="left"))
        assert b[0] == 0 and b[-1] == P


# ---- downstream consumers: the reference's filter_view / histogram -------

def test_consumer_oracles_match_reference(golden_cases):
    c = golden_cases["seed500"]
    g = np.load(GOLDEN / "consumers_seed500.npz")
    n = 500
    payload, lens = c["payload"], c["lengths"]
    # raw and normalised histograms (store.py:342-381)
    h = orc.np_histogram(payload)
    first = int(g["hist_raw_first"][0])
    assert np.array_equal(h[first + 128: first + 128 + len(g["hist_raw_counts"])], g["hist_raw_counts"])
    assert h.sum() == g["hist_raw_counts"].sum()
    hn = orc.np_hist_normalized(payload, 0, n, lens)
    first = int(g["hist_norm_first"][0])
    assert np.array_equal(hn[first + 12800: first + 12800 + len(g["hist_norm_counts"])], g["hist_norm_counts"])
    assert hn.sum() == g["hist_norm_counts"].sum() == payload.size
    # normalised filter windows (graph.py:91-101)
    for k in range(5):
        lo, hi = g[f"filter{k}_bounds"]
        idx, sc, deg = orc.np_filter_normalized(payload, 0, n, lens, lo, hi)
        assert idx.size == int(g[f"filter{k}_count"][0])
        assert np.array_equal(deg, g[f"filter{k}_degree"])
        if f"filter{k}_edges" in g:
            rows = orc.np_rows_of(idx, n)
            cols = orc.np_cols_of(idx, n, rows)
            assert np.array_equal(np.stack([rows, cols], 1), g[f"filter{k}_edges"].astype(np.int64))


def test_oracle_reproduces_the_reference_c2_payload():
    """configs[1] at full size: the C oracle's 199,990,000 bytes hash to the digest of the payload the UNMODIFIED
    reference engine produced (tests/golden/c2_reference_digest.json, made by make_golden_c2_digest.py), and the
    statistics equal its ComputeStats."""
    import hashlib
    import json
    import os
    from conftest import GOLDEN
    from paper_2509_01654_b200 import synth

    gold = json.loads((GOLDEN / "c2_reference_digest.json").read_text())
    ids, lens, sch = synth.config_store("C2")
    assert synth.store_digest(ids, lens) == gold["store_digest"] and list(sch) == gold["scheme"]
    n = len(lens)
    P = n * (n - 1) // 2
    sim = orc.similarity_matrix(sch[0], sch[1], int(ids.max()) + 1)
    payload, ssum, smin, smax = orc.c_score_range(ids.astype(np.int32), lens.astype(np.int32), sim, sch[2], n, 0, P,
                                                  threads=len(os.sched_getaffinity(0)))
    assert payload.size == gold["edges"] == P
    assert hashlib.blake2b(payload.tobytes(), digest_size=16).hexdigest() == gold["payload_blake2b_128"]
    assert (smin, smax) == (gold["min"], gold["max"]) and ssum / P == gold["mean"]
