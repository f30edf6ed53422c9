"""Host logic of the drop-in boundary, CPU only: types, preflight messages, plan
validation, packing, shard arithmetic -- mirroring reference tests/test_engine.py."""
import numpy as np
import pytest

import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import sharding, synth
from paper_2509_01654_b200.engine import pack_words, similarity_table
from oracle import nw_oracle as orc


class CollectSink:
    def __init__(self):
        self.chunks, self.aborted = [], False

    def write(self, data):
        self.chunks.append(bytes(data))

    def abort(self):
        self.aborted = True


def test_preflight_ok_returns_max_length():
    words = synth.make_words(10, seed=1, min_len=3, max_len=20)
    assert nw.preflight_range_check(words, nw.ScoringScheme(1, -1, -1)) == max(len(w.phonemes) for w in words)


def test_preflight_overflow_messages():
    words = [nw.EncodedWord("long", "x", tuple([0] * 70), 1.0), nw.EncodedWord("late", "y", (0, 1), 1.0)]
    with pytest.raises(nw.DataError, match="-280"):
        nw.preflight_range_check(words, nw.ScoringScheme(1, -1, -2))
    with pytest.raises(nw.DataError, match="> 127"):
        nw.preflight_range_check([nw.EncodedWord("w", "x", tuple([0] * 20), 1.0)], nw.ScoringScheme(10, -1, -1))
    with pytest.raises(ValueError):
        nw.preflight_range_check([], nw.ScoringScheme())


def test_plan_validation_and_chunks():
    with pytest.raises(ValueError):
        nw.ComputePlan(n=1)
    with pytest.raises(ValueError):
        nw.ComputePlan(n=5, chunk_size=0)
    with pytest.raises(ValueError):
        nw.ComputePlan(n=5, worker_count=0)
    chunks = list(nw.ComputePlan(n=123, chunk_size=97).chunks())
    assert chunks[0][0] == 0 and chunks[-1][1] == nw.num_edges(123)
    assert all(a[1] == b[0] for a, b in zip(chunks, chunks[1:]))


def test_argument_checks_run_before_any_device_work():
    words = synth.make_words(5, seed=0)
    with pytest.raises(ValueError, match="plan is for"):
        nw.compute_all_pairs(words, nw.ScoringScheme(), CollectSink(), nw.ComputePlan(n=6))
    with pytest.raises(ValueError, match="scheme"):
        nw.compute_all_pairs(words, nw.ScoringScheme(), CollectSink(),
                             nw.ComputePlan(n=5, scheme=nw.ScoringScheme(2)))


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sink = CollectSink()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        nw.compute_all_pairs(synth.make_words(5, seed=0), nw.ScoringScheme(), sink)
    assert not sink.chunks and sink.aborted      # the sink is told, so a writer can mark its store incomplete


def test_scheme_semantics():
    s = nw.ScoringScheme(1, -1, -1, overrides={(1, 2): 1})
    assert s.similarity(2, 1) == 1 and s.similarity(1, 1) == 1 and s.similarity(0, 1) == -1
    assert (s.min_similarity, s.max_similarity) == (-1, 1)
    with pytest.raises(ValueError):
        nw.ScoringScheme(overrides={(1, 2): 1, (2, 1): 0})
    t = similarity_table(s, 4)
    assert t[1, 2] == t[2, 1] == 1 and t[0, 0] == 1 and t[0, 3] == -1
    assert np.array_equal(t, orc.similarity_matrix(1, -1, 4, {(1, 2): 1}))


def test_pack_words_matches_reference_layout(golden_cases):
    c = golden_cases["seed9"]
    words = synth.make_words(30, seed=9, alphabet=8, min_len=1, max_len=9)
    ids, lens = pack_words(words)
    assert np.array_equal(ids, c["ids"]) and np.array_equal(lens, c["lengths"])
    with pytest.raises(ValueError):
        pack_words([nw.EncodedWord("e", "e", (), 1.0), nw.EncodedWord("f", "f", (1,), 1.0)])


def test_triangle_scalars(golden_triangle):
    t = golden_triangle
    for n in (4, 300, 10 ** 5, 10 ** 7):
        idx, rows, cols = t[f"n{n}_idx"], t[f"n{n}_rows"], t[f"n{n}_cols"]
        for k in range(0, len(idx), max(1, len(idx) // 300)):
            r = nw.row_of(int(idx[k]), n)
            assert r == rows[k] and nw.col_of(int(idx[k]), n, r) == cols[k]
            assert nw.index_of(r, int(cols[k]), n) == idx[k]
    assert nw.num_edges(600_000) == 179_999_700_000


def test_equal_work_bounds_match_oracle_and_balance():
    ids, lens, _ = synth.config_store("C2")
    for parts in (1, 2, 4, 8):
        b = sharding.equal_work_bounds(lens, parts)
        assert np.array_equal(b, orc.np_equal_work_bounds(lens, parts))
        assert b[0] == 0 and b[-1] == nw.num_edges(len(lens)) and (np.diff(b) >= 0).all()
    b = sharding.equal_work_bounds(lens, 8)
    lens32 = lens.astype(np.int32)
    work = [orc.cells_in_range(lens32, len(lens), int(b[g]), int(b[g + 1])) for g in range(8)]
    assert sum(work) == synth.total_cells(lens)
    assert max(work) - min(work) <= 2 * int(lens.max()) ** 2      # equal to within one pair's cells
    # a frequency-ordered (short words first) store: equal pairs would be badly unequal work
    order = np.argsort(lens, kind="stable")
    b2 = sharding.equal_work_bounds(lens[order], 8)
    work2 = [orc.cells_in_range(lens32[order], len(lens), int(b2[g]), int(b2[g + 1])) for g in range(8)]
    assert max(work2) - min(work2) <= 2 * int(lens.max()) ** 2


def test_synth_generators_are_frozen(golden_samples):
    meta, _ = golden_samples
    ids, lens, sch = synth.config_store("C5")
    assert sch == (2, -1, -3) and int(lens.max()) <= 21
    assert synth.store_digest(ids, lens) == meta["C5"]["store_digest"]
    w = synth.as_encoded_words(ids[:50], lens[:50])
    assert nw.preflight_range_check(w, nw.ScoringScheme(*sch)) <= 21
