"""Parity of the CUDA path (through the C ABI) with the oracle, the reference's golden
vectors and the reference tests' own cases.  Bit-exact: this is integer/byte work."""
import hashlib
import json

import numpy as np
import pytest

import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import _native, synth
from paper_2509_01654_b200.engine import NwapContext, device_rows_cols
from oracle import nw_oracle as orc
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FAST = ["packed", "packed3", "packed_sym"]
ALL = ["packed", "packed3", "packed_sym", "simple"]


def _allowed(variants, scheme):
    """packed_sym (2 DPX + IADD3 cell) needs match >= mismatch and no overrides."""
    ok = scheme.match >= scheme.mismatch and not scheme.overrides
    return [v for v in variants if v != "packed_sym" or ok]


@pytest.mark.parametrize("n", [5119, 5120, 5121, 10241])
def test_strip_boundary_sizes(n):
    """Vocabulary sizes around whole strips of the tile kernel (5120 columns): ragged last strip of 1 column,
    exactly full strips, one column over; every byte and the statistics against the oracle, plus a range that
    starts and ends mid-row next to a strip boundary."""
    rng = np.random.default_rng(n)
    lens = np.clip(np.rint(rng.normal(8.5, 2.8, size=n)), 1, 24).astype(np.uint8)
    ids = rng.integers(0, 40, size=(n, 24)).astype(np.uint8)
    scheme = nw.ScoringScheme(1, -1, -2)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P, threads=len(__import__("os").sched_getaffinity(0)))
    with NwapContext(ids, lens, scheme) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        st = ctx.score_range(0, P, out)
        assert np.array_equal(out.cpu().numpy(), ref)
        assert st[:4] == (rsum, rmin, rmax, P)
        s = nw.index_of(7, 5118, n)
        e = nw.index_of(3000, n - 2, n) if n > 3002 else P
        got, st2 = _score(ctx, s, e, "auto", offset=5)
        assert np.array_equal(got, ref[s:e])
        sub = ref[s:e].astype(np.int64)
        assert st2[:4] == (int(sub.sum()), int(sub.min()), int(sub.max()), e - s)


class CollectSink:
    def __init__(self, fail_at=None):
        self.chunks, self.aborted, self.fail_at = [], False, fail_at

    def write(self, data):
        if self.fail_at is not None and len(self.chunks) >= self.fail_at:
            raise OSError("disk full")
        self.chunks.append(bytes(data))

    def abort(self):
        self.aborted = True

    @property
    def payload(self):
        return b"".join(self.chunks)


def _scheme(case):
    m, x, g = case["scheme"]
    return nw.ScoringScheme(m, x, g, overrides={(a, b): v for a, b, v in case.get("overrides", [])})


def _score(ctx, start, end, variant, offset=0, want_hist=False):
    buf = torch.full((end - start + offset + 64,), 0x55, dtype=torch.int8, device="cuda")
    out = buf[offset:]
    st = ctx.score_range(start, end, out, want_hist=want_hist, variant=variant)
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    # nothing outside [offset, offset + end - start) may be touched
    assert (host[:offset] == 0x55).all() and (host[offset + end - start:] == 0x55).all()
    return host[offset: offset + end - start], st


def _oracle(ids, lens, scheme, start, end, threads=1):
    m, x, g = scheme.match, scheme.mismatch, scheme.gap
    sim = orc.similarity_matrix(m, x, int(ids.max()) + 1, dict(scheme.overrides))
    return orc.c_score_range(ids.astype(np.int32), lens.astype(np.int32), sim, g, len(lens), start, end,
                             threads=threads)


def test_library_is_the_cuda_one():
    assert _native.lib().nwap_device_count() >= 1
    assert torch.cuda.get_device_capability(0)[0] >= 10


# ---- the reference tests' own cases (tests/test_engine.py) --------------------------------

def test_two_word_payload_is_single_byte():
    words = [nw.EncodedWord("puissance", "x", (0, 18, 16, 11, 26, 11), 1.0),
             nw.EncodedWord("nuance", "y", (29, 18, 26, 11), 1.0)]
    sink = CollectSink()
    nw.compute_all_pairs(words, nw.ScoringScheme(1, -1, -2), sink)
    assert sink.payload == b"\xfe"


def test_identical_words_score_their_length():
    words = [nw.EncodedWord(f"w{i}", f"i{i}", (3, 1, 4, 1, 5), 1.0) for i in range(6)]
    sink = CollectSink()
    stats = nw.compute_all_pairs(words, nw.ScoringScheme(), sink)
    assert sink.payload == bytes([5]) * 15
    assert stats.min_score == stats.max_score == 5 and stats.mean_score == 5.0 and stats.edges_written == 15


def test_scheme_overrides_respected():
    words = [nw.EncodedWord("a", "a", (0, 1), 1.0), nw.EncodedWord("b", "b", (0, 2), 1.0)]
    sink = CollectSink()
    nw.compute_all_pairs(words, nw.ScoringScheme(1, -1, -1, overrides={(1, 2): 1}), sink)
    assert sink.payload == bytes([2])


@pytest.mark.parametrize("chunk_size", [7, 64, 1024, 10 ** 6])
def test_payload_independent_of_partitioning(golden_cases, chunk_size):
    c = golden_cases["seed4"]
    words = synth.make_words(40, seed=4, alphabet=10)
    scheme = nw.ScoringScheme(2, -1, -2)
    sink = CollectSink()
    plan = nw.ComputePlan(n=40, chunk_size=chunk_size, worker_count=2, scheme=scheme)
    nw.compute_all_pairs(words, scheme, sink, plan)
    assert sink.payload == c["payload"].tobytes()
    assert all(len(ch) <= chunk_size for ch in sink.chunks)


def test_stats_are_exact(golden_cases):
    c = golden_cases["seed11"]
    sink = CollectSink()
    stats = nw.compute_all_pairs(synth.make_words(25, seed=11), nw.ScoringScheme(), sink)
    scores = np.frombuffer(sink.payload, dtype=np.int8)
    assert np.array_equal(scores, c["payload"])
    assert stats.edges_written == 300 and stats.min_score == c["min"] and stats.max_score == c["max"]
    assert stats.mean_score == c["mean"] == float(scores.astype(np.int64).mean())


def test_sink_failure_aborts():
    sink = CollectSink(fail_at=1)
    with pytest.raises(OSError):
        nw.compute_all_pairs(synth.make_words(40, seed=4), nw.ScoringScheme(), sink, nw.ComputePlan(n=40, chunk_size=100))
    assert sink.aborted


def test_host_pipeline_begin_wait_and_context_cycle():
    """The split host-destination call (two host slabs alternating, as compute_all_pairs drives it), the
    create -> score -> destroy cycle served from the per-device cache, and nwap_trim()."""
    ids, lens = synth.french_shaped(3000)
    scheme = nw.ScoringScheme(1, -1, -2)
    P = nw.num_edges(3000)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P, threads=4)
    slabs = [torch.empty(1 << 20, dtype=torch.int8).pin_memory() for _ in range(2)]
    for cycle in range(3):
        with NwapContext(ids, lens, scheme) as ctx:
            ranges = [(s, min(P, s + (1 << 20))) for s in range(0, P, 1 << 20)]
            got = np.empty(P, dtype=np.int8)
            tot = 0
            ctx.score_range_host_begin(*ranges[0], slabs[0])
            with pytest.raises(ValueError, match="already in flight"):
                ctx.score_range_host_begin(*ranges[0], slabs[1])
            for k, (s, e) in enumerate(ranges):
                st = ctx.score_range_host_wait()
                if k + 1 < len(ranges):
                    ctx.score_range_host_begin(*ranges[k + 1], slabs[(k + 1) & 1])
                got[s:e] = slabs[k & 1].numpy()[: e - s]
                tot += st[0]
                assert st[3] == e - s
            assert np.array_equal(got, ref) and tot == rsum
            with pytest.raises(ValueError, match="no host-destination call"):
                ctx.score_range_host_wait()
        if cycle == 1:
            _native.lib().nwap_trim()          # the next context re-creates its pipeline


def test_entry_point_with_many_slabs_matches_oracle():
    """compute_all_pairs with more than two staging slabs in flight order (sink sees index order)."""
    words = synth.make_words(1500, seed=77, alphabet=30, min_len=1, max_len=12)
    scheme = nw.ScoringScheme(1, -1, -2)
    sink = CollectSink()
    plan = nw.ComputePlan(n=1500, chunk_size=1000, scheme=scheme)
    import paper_2509_01654_b200.engine as eng
    old = eng._SLAB_BYTES
    eng._SLAB_BYTES = 200_000                   # 6 slabs of 200 chunks
    try:
        stats = nw.compute_all_pairs(words, scheme, sink, plan)
    finally:
        eng._SLAB_BYTES = old
    wid, wl = synth.store_from_words(words)
    ref, rsum, rmin, rmax = _oracle(wid, wl, scheme, 0, nw.num_edges(1500), threads=4)
    assert sink.payload == ref.tobytes()
    assert (stats.edges_written, stats.min_score, stats.max_score) == (len(ref), rmin, rmax)
    assert stats.mean_score == rsum / len(ref)
    assert all(len(c) == 1000 for c in sink.chunks[:-1])


class RetainingSink:
    """The reference tests' own sink shape (tests/test_engine.py:14-31, test_acceptance.py `Collect`):
    keeps the object it is handed and joins later."""

    def __init__(self):
        self.chunks, self.aborted = [], False

    def write(self, data):
        self.chunks.append(data)

    def abort(self):
        self.aborted = True


class ViewSink:
    """Opt-in zero-copy sink: consumes the transient view inside the call."""

    def __init__(self):
        self.h = hashlib.blake2b(digest_size=16)
        self.n = 0
        self.types = set()

    def write(self, data):                     # never called when write_view exists
        raise AssertionError("write() called on a sink that defines write_view()")

    def write_view(self, view):
        self.types.add(type(view))
        self.h.update(view)
        self.n += len(view)

    def abort(self):
        raise AssertionError("abort")


def test_sink_gets_immutable_bytes_that_survive_slab_reuse():
    """A sink that KEEPS what it is handed (as the reference's test sinks do) must end up with the right payload
    when the job spans more than two staging slabs and when two runs follow each other: write() receives
    bytes objects, never views into the recycled pinned slabs; write_view() is the opt-in transient path."""
    words = synth.make_words(1500, seed=77, alphabet=30, min_len=1, max_len=12)
    scheme = nw.ScoringScheme(1, -1, -2)
    plan = nw.ComputePlan(n=1500, chunk_size=1000, scheme=scheme)
    wid, wl = synth.store_from_words(words)
    ref, *_ = _oracle(wid, wl, scheme, 0, nw.num_edges(1500), threads=4)
    words2 = synth.make_words(1500, seed=78, alphabet=30, min_len=1, max_len=12)
    wid2, wl2 = synth.store_from_words(words2)
    ref2, *_ = _oracle(wid2, wl2, scheme, 0, nw.num_edges(1500), threads=4)
    import paper_2509_01654_b200.engine as eng
    old = eng._SLAB_BYTES
    eng._SLAB_BYTES = 200_000                   # 6 slabs: every staging slab is reused three times
    try:
        a, b, v = RetainingSink(), RetainingSink(), ViewSink()
        nw.compute_all_pairs(words, scheme, a, plan)
        nw.compute_all_pairs(words2, scheme, b, plan)      # recycles the first run's slabs
        nw.compute_all_pairs(words, scheme, v, plan)
    finally:
        eng._SLAB_BYTES = old
    assert all(type(c) is bytes for c in a.chunks + b.chunks)
    assert b"".join(a.chunks) == ref.tobytes()
    assert b"".join(b.chunks) == ref2.tobytes()
    assert v.types == {memoryview} and v.n == len(ref)
    assert v.h.hexdigest() == hashlib.blake2b(ref.tobytes(), digest_size=16).hexdigest()


def test_huge_chunk_size_is_one_piece_and_pins_only_the_job():
    """ComputePlan(chunk_size=2**31) on a tiny job: one write of the whole payload, no 2 GiB pinned slab."""
    import paper_2509_01654_b200.engine as eng
    words = synth.make_words(40, seed=4, alphabet=10)
    scheme = nw.ScoringScheme(2, -1, -2)
    sink = RetainingSink()
    eng.trim()
    nw.compute_all_pairs(words, scheme, sink, nw.ComputePlan(n=40, chunk_size=2 ** 31, scheme=scheme))
    assert [len(c) for c in sink.chunks] == [780]
    assert sum(t.numel() for have in eng._STAGING.values() for t in have) <= 1 << 20


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_entry_point_shares_slabs_between_contexts(devices):
    """The single-process multi-GPU path of compute_all_pairs (slab k -> device k mod G), exercised with
    several contexts on the one GPU this box has: same payload, statistics and chunking for any G."""
    words = synth.make_words(1200, seed=5, alphabet=25, min_len=1, max_len=14)
    scheme = nw.ScoringScheme(2, -1, -2)
    plan = nw.ComputePlan(n=1200, chunk_size=4096, scheme=scheme)
    import paper_2509_01654_b200.engine as eng
    old = eng._SLAB_BYTES
    eng._SLAB_BYTES = 100_000                   # 30 slabs of 24 chunks
    try:
        sink = CollectSink()
        stats = nw.compute_all_pairs(words, scheme, sink, plan, devices=devices)
        bad = CollectSink(fail_at=40)
        with pytest.raises(OSError):
            nw.compute_all_pairs(words, scheme, bad, plan, devices=devices)
        assert bad.aborted
    finally:
        eng._SLAB_BYTES = old
    wid, wl = synth.store_from_words(words)
    ref, rsum, rmin, rmax = _oracle(wid, wl, scheme, 0, nw.num_edges(1200), threads=4)
    assert sink.payload == ref.tobytes()
    assert (stats.edges_written, stats.min_score, stats.max_score) == (len(ref), rmin, rmax)
    assert stats.mean_score == rsum / len(ref)
    assert all(len(c) == 4096 for c in sink.chunks[:-1])
    with pytest.raises(ValueError, match="at least one GPU"):
        nw.compute_all_pairs(words, scheme, CollectSink(), plan, devices=[])


def test_errors_surface_as_reference_exceptions():
    with pytest.raises(nw.DataError, match="-280"):
        nw.compute_all_pairs([nw.EncodedWord("l", "x", tuple([0] * 70), 1.0), nw.EncodedWord("s", "y", (0, 1), 1.0)],
                             nw.ScoringScheme(1, -1, -2), CollectSink())
    ids = np.zeros((3, 4), dtype=np.uint8)
    with pytest.raises(ValueError, match="empty"):
        NwapContext(ids, np.array([2, 0, 1], dtype=np.uint8), nw.ScoringScheme())
    with pytest.raises(nw.DataError):
        NwapContext(np.zeros((2, 70), dtype=np.uint8), np.array([70, 2], dtype=np.uint8), nw.ScoringScheme(1, -1, -2))
    with NwapContext(np.zeros((4, 40), dtype=np.uint8), np.full(4, 40, dtype=np.uint8), nw.ScoringScheme()) as ctx:
        out = torch.empty(6, dtype=torch.int8, device="cuda")
        with pytest.raises(ValueError, match="packed kernel"):
            ctx.score_range(0, 6, out, variant="packed")
        with pytest.raises(ValueError):
            ctx.score_range(0, 7, torch.empty(7, dtype=torch.int8, device="cuda"))


# ---- golden engine payloads, every kernel variant ------------------------------------------

@pytest.mark.parametrize("name", ["seed9", "seed4", "seed11", "seed30", "seed500", "gap0", "gappos",
                                  "mis_gt_match", "long40", "override"])
def test_golden_engine_cases(golden_cases, name):
    c = golden_cases[name]
    scheme = _scheme(c)
    n = len(c["lengths"])
    P = nw.num_edges(n)
    with NwapContext(c["ids"], c["lengths"], scheme) as ctx:
        # sparse overrides run on the packed kernel too; q > 32 only on the generic one
        variants = ["simple"] if ctx.max_len > 32 else (["packed3", "simple"] if c.get("overrides") else ALL)
        for v in _allowed(variants, scheme) + ["auto"]:
            got, st = _score(ctx, 0, P, v, want_hist=True)
            assert np.array_equal(got, c["payload"]), (name, v)
            ssum, smin, smax, scount, hist = st
            assert (smin, smax, scount) == (c["min"], c["max"], P)
            assert ssum / P == c["mean"]
            assert np.array_equal(hist, orc.np_histogram(c["payload"]))
            assert hashlib.blake2b(got.tobytes(), digest_size=8).hexdigest() == c["digest"]


@pytest.mark.parametrize("variant", ALL)
def test_arbitrary_subranges_and_alignments(golden_cases, variant):
    c = golden_cases["seed500"]
    n, P = 500, nw.num_edges(500)
    rng = np.random.default_rng(3)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        cases = [(0, 1), (P - 1, P), (0, 499), (498, 500), (499, 499 + 498), (P - 3, P), (7, 7)]
        for _ in range(40):
            s = int(rng.integers(0, P))
            e = int(min(P, s + rng.integers(1, 30_000)))
            cases.append((s, e))
        for k, (s, e) in enumerate(cases):
            got, st = _score(ctx, s, e, variant, offset=k % 17)
            assert np.array_equal(got, c["payload"][s:e]), (s, e)
            if e > s:
                ref = c["payload"][s:e].astype(np.int64)
                assert st[:4] == (int(ref.sum()), int(ref.min()), int(ref.max()), e - s)
            else:
                assert st[:4] == (0, 127, -128, 0)


@pytest.mark.parametrize("variant", FAST)
def test_length_extremes(variant):
    rng = np.random.default_rng(11)
    for n, lo, hi, sch in [(2, 1, 1, (1, -1, -1)), (3, 32, 32, (1, -1, -2)), (700, 1, 32, (1, -1, -2)),
                           (2100, 1, 3, (2, -1, -3)), (2060, 30, 32, (1, -1, -1)), (4100, 1, 16, (3, -2, -4))]:
        lens = rng.integers(lo, hi + 1, size=n).astype(np.uint8)
        ids = rng.integers(0, 5, size=(n, hi)).astype(np.uint8)
        scheme = nw.ScoringScheme(*sch)
        P = nw.num_edges(n)
        ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P, threads=4)
        with NwapContext(ids, lens, scheme) as ctx:
            got, st = _score(ctx, 0, P, variant)
            assert np.array_equal(got, ref), (n, lo, hi)
            assert st[:4] == (rsum, rmin, rmax, P)


def test_random_schemes_all_variants():
    rng = np.random.default_rng(2024)
    for trial in range(12):
        q = int(rng.integers(2, 33))
        while True:
            m, x, g = int(rng.integers(-3, 5)), int(rng.integers(-4, 5)), int(rng.integers(-4, 4))
            if min(0, 2 * q * g, q * min(m, x)) >= -128 and max(0, 2 * q * g, q * max(m, x)) <= 127:
                break
        n = int(rng.integers(40, 400))
        lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
        lens[0] = q
        ids = rng.integers(0, int(rng.integers(2, 41)), size=(n, q)).astype(np.uint8)
        scheme = nw.ScoringScheme(m, x, g)
        P = nw.num_edges(n)
        ref, *_ = _oracle(ids, lens, scheme, 0, P)
        with NwapContext(ids, lens, scheme) as ctx:
            for v in _allowed(ALL, scheme) + ["auto"]:
                got, _ = _score(ctx, 0, P, v)
                assert np.array_equal(got, ref), (trial, v, (m, x, g), q)
            if m < x:
                with pytest.raises(ValueError, match="packed_sym"):
                    ctx.score_range(0, 10, torch.empty(10, dtype=torch.int8, device="cuda"), variant="packed_sym")


def test_sparse_override_schemes_on_the_packed_kernel():
    """ScoringScheme.overrides: random sparse override sets must give the same bytes on the packed sparse-override
    kernel (at most 2 partners per symbol: NWAP_MAX_OV), the generic kernel and the oracle; a denser table is
    refused by the sparse-override cell and served by the table-driven / generic one."""
    rng = np.random.default_rng(77)
    for trial in range(12):
        q = int(rng.integers(4, 25))
        K = int(rng.integers(3, 41)) if trial < 10 else (128, 97)[trial - 10]    # the partner table's largest alphabets
        while True:
            m, x, g = int(rng.integers(0, 4)), int(rng.integers(-4, 1)), int(rng.integers(-4, 0))
            ov = {}
            for _ in range(int(rng.integers(1, 6))):
                a_, b_ = int(rng.integers(0, K)), int(rng.integers(0, K))
                ov[(min(a_, b_), max(a_, b_))] = int(rng.integers(-4, 5))
            vals = [m, x, *ov.values()]
            if min(0, 2 * q * g, q * min(vals)) >= -128 and max(0, 2 * q * g, q * max(vals)) <= 127:
                break
        n = int(rng.integers(300, 2600))
        lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
        lens[0] = q
        ids = rng.integers(0, K, size=(n, q)).astype(np.uint8)
        scheme = nw.ScoringScheme(m, x, g, overrides=ov)
        P = nw.num_edges(n)
        ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P, threads=4)
        partners = {}
        for (a_, b_), val in ov.items():
            if val != (m if a_ == b_ else x):
                partners.setdefault(a_, set()).add(b_)
                partners.setdefault(b_, set()).add(a_)
        sparse = all(len(v_) <= 2 for v_ in partners.values())
        with NwapContext(ids, lens, scheme) as ctx:
            for v in ("auto", "packed3", "simple"):
                if v == "packed3" and not sparse:
                    with pytest.raises(ValueError, match="packed kernel"):
                        _score(ctx, 0, P, v)
                    continue
                got, st = _score(ctx, 0, P, v, want_hist=(trial % 2 == 0))
                assert np.array_equal(got, ref), (trial, v, (m, x, g), ov)
                assert st[:4] == (rsum, rmin, rmax, P)
    # dense table: every pair overridden
    K, n, q = 6, 200, 8
    ids = rng.integers(0, K, size=(n, q)).astype(np.uint8)
    lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
    ov = {(a, b): int((a * 7 + b * 3) % 5 - 2) for a in range(K) for b in range(a, K)}
    scheme = nw.ScoringScheme(1, -1, -2, overrides=ov)
    ref, *_ = _oracle(ids, lens, scheme, 0, nw.num_edges(n))
    with NwapContext(ids, lens, scheme) as ctx:
        got, _ = _score(ctx, 0, nw.num_edges(n), "auto")
        assert np.array_equal(got, ref)
        with pytest.raises(ValueError, match="packed kernel"):
            ctx.score_range(0, 10, torch.empty(10, dtype=torch.int8, device="cuda"), variant="packed3")


def test_dense_similarity_tables_on_the_packed_kernel():
    """Dense override tables (every pair has its own value) run on the packed kernel's table-driven flavour for every
    alphabet the uint8 word store admits (K <= 256; the K x K table is dynamic shared memory): same bytes and statistics
    as the generic kernel and the oracle."""
    rng = np.random.default_rng(314)
    for trial, (K, q, n) in enumerate([(6, 8, 300), (40, 24, 2500), (128, 16, 1200), (17, 32, 700), (3, 1, 50), (40, 12, 5200)]):
        while True:
            g = int(rng.integers(-4, 1))
            lo_s, hi_s = sorted(int(x) for x in rng.integers(-4, 5, size=2))
            if min(0, 2 * q * g, q * lo_s) >= -128 and max(0, 2 * q * g, q * hi_s) <= 127 and lo_s < hi_s:
                break
        ov = {(a, b): int(rng.integers(lo_s, hi_s + 1)) for a in range(K) for b in range(a, K)}
        lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
        lens[0] = q
        ids = rng.integers(0, K, size=(n, q)).astype(np.uint8)
        ids[1, 0] = K - 1
        scheme = nw.ScoringScheme(ov[(0, 0)], ov[(0, 1)] if K > 1 else 0, g, overrides=ov)
        P = nw.num_edges(n)
        ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P, threads=8)
        with NwapContext(ids, lens, scheme) as ctx:
            for v in ("auto", "packed_tab", "simple"):
                got, st = _score(ctx, 0, P, v, want_hist=(trial % 2 == 0), offset=trial)
                assert np.array_equal(got, ref), (trial, v, K, q, g)
                assert st[:4] == (rsum, rmin, rmax, P)
            s, e = P // 3, P // 3 + min(P // 2, 70_001)
            got, st = _score(ctx, s, e, "packed_tab", offset=3)
            assert np.array_equal(got, ref[s:e])
            if K >= 17:          # certainly more than 3 override partners per symbol: the compare-based cells refuse
                with pytest.raises(ValueError, match="packed kernel"):
                    ctx.score_range(0, 10, torch.empty(10, dtype=torch.int8, device="cuda"), variant="packed3")
    # a uniform scheme has no table: packed_tab is refused
    with NwapContext(ids, lens, nw.ScoringScheme(1, -1, -1)) as ctx:
        with pytest.raises(ValueError, match="packed_tab"):
            ctx.score_range(0, 10, torch.empty(10, dtype=torch.int8, device="cuda"), variant="packed_tab")
    # 128 < K <= 256: still the table-driven cell (one CTA per SM: the table takes up to 64 KB)
    for K, n, q in ((200, 900, 6), (256, 700, 9)):
        ids = rng.integers(0, K, size=(n, q)).astype(np.uint8)
        ids[0, 0] = K - 1
        lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
        ov = {(a, b): int((a * 7 + b * 3) % 5 - 2) for a in range(K) for b in range(a, K)}
        scheme = nw.ScoringScheme(1, -1, -2, overrides=ov)
        ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, nw.num_edges(n), threads=4)
        with NwapContext(ids, lens, scheme) as ctx:
            for v in ("auto", "packed_tab", "simple"):
                got, st = _score(ctx, 0, nw.num_edges(n), v)
                assert np.array_equal(got, ref), (K, v)
                assert st[:4] == (rsum, rmin, rmax, nw.num_edges(n))
    # words over 32 symbols with an override scheme: the wide build of the table-driven cell (was: the generic kernel)
    K, n, q = 12, 300, 40
    ids = rng.integers(0, K, size=(n, q)).astype(np.uint8)
    lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
    lens[0] = q
    scheme = nw.ScoringScheme(1, -1, -1, overrides={(0, 1): 0, (2, 3): 1})
    ref, *_ = _oracle(ids, lens, scheme, 0, nw.num_edges(n))
    with NwapContext(ids, lens, scheme) as ctx:
        for v in ("auto", "packed_tab", "simple"):
            got, _ = _score(ctx, 0, nw.num_edges(n), v)
            assert np.array_equal(got, ref), v
        with pytest.raises(ValueError, match="packed kernel"):      # the compare-based override cell stays at 32 symbols
            ctx.score_range(0, 10, torch.empty(10, dtype=torch.int8, device="cuda"), variant="packed3")


# ---- BASELINE.json configs -------------------------------------------------------------------

def test_c1_full_config_through_entry_point(golden_samples):
    meta, _ = golden_samples
    ref = np.load(GOLDEN / "c1.npz")["payload"]
    ids, lens, sch = synth.config_store("C1")
    words = synth.as_encoded_words(ids, lens)
    sink = CollectSink()
    stats = nw.compute_all_pairs(words, nw.ScoringScheme(*sch), sink)
    assert sink.payload == ref.tobytes()
    assert (stats.min_score, stats.max_score, stats.mean_score) == (meta["C1"]["min"], meta["C1"]["max"], meta["C1"]["mean"])
    assert hashlib.blake2b(sink.payload, digest_size=8).hexdigest() == meta["C1"]["digest"]


def test_c2_every_byte_against_oracle(golden_samples):
    """configs[1]: 20,000 words, all 199,990,000 pairs bit-exact vs the CPU oracle."""
    ids, lens, sch = synth.config_store("C2")
    scheme = nw.ScoringScheme(*sch)
    n = len(lens)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P, threads=0 or len(__import__("os").sched_getaffinity(0)))
    with NwapContext(ids, lens, scheme) as ctx:
        for v in ALL:
            out = torch.empty(P, dtype=torch.int8, device="cuda")
            st = ctx.score_range(0, P, out, want_hist=True, variant=v)
            got = out.cpu().numpy()
            assert np.array_equal(got, ref), v
            assert st[:4] == (rsum, rmin, rmax, P)
            assert np.array_equal(st[4], orc.np_histogram(ref))
        # host-destination pipeline (the e2e call) and the independent statistics kernel
        host = torch.empty(P, dtype=torch.int8).pin_memory()
        st = ctx.score_range_host(0, P, host, want_hist=True)
        assert np.array_equal(host.numpy(), ref) and st[:4] == (rsum, rmin, rmax, P)
        # ... and the payload the UNMODIFIED reference engine produced for this config (its digest and ComputeStats)
        gold = json.loads((GOLDEN / "c2_reference_digest.json").read_text())
        assert hashlib.blake2b(host.numpy().tobytes(), digest_size=16).hexdigest() == gold["payload_blake2b_128"]
        assert (st[1], st[2], st[0] / P) == (gold["min"], gold["max"], gold["mean"])
        ps = ctx.payload_stats(out)
        assert ps[:4] == (rsum, rmin, rmax, P) and np.array_equal(ps[4], orc.np_histogram(ref))
        # equal-work shards written independently reproduce the payload (multi-GPU path, one GPU)
        bounds = ctx.equal_work_bounds(8)
        from paper_2509_01654_b200 import sharding
        assert np.array_equal(bounds, sharding.equal_work_bounds(lens, 8))
        whole = torch.zeros(P, dtype=torch.int8, device="cuda")
        tot = 0
        for g in range(8):
            s, e = int(bounds[g]), int(bounds[g + 1])
            stg = ctx.score_range(s, e, whole[s:e])
            tot += stg[0]
        assert np.array_equal(whole.cpu().numpy(), ref) and tot == rsum


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_sampled_ranges_of_big_configs(golden_samples, cfg):
    """configs[2..4]: ranges scored by the reference's _score_range (golden) byte for byte."""
    meta, arrays = golden_samples
    m = meta[cfg]
    ids, lens, sch = synth.config_store(cfg)
    assert synth.store_digest(ids, lens) == m["store_digest"]
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        for k, r in enumerate(m["ranges"]):
            for v in ALL:
                got, st = _score(ctx, r["start"], r["end"], v, offset=k)
                assert np.array_equal(got, arrays[f"{cfg}_{k}"]), (cfg, k, v)
                assert st[:3] == (r["sum"], r["min"], r["max"])
        # equal-work bounds agree between the library and the host mirror
        from paper_2509_01654_b200 import sharding
        assert np.array_equal(ctx.equal_work_bounds(8), sharding.equal_work_bounds(lens, 8))
        assert ctx.cells_in_range(0, ctx.num_edges) == m["total_cells"]


def test_c3_every_byte_against_the_reference_itself():
    """configs[2] at full size: the 8 equal-work shards, scored independently (what 8 ranks would write), hash to the
    per-shard digests of the payload the UNMODIFIED reference engine produced for the same 100,000 words
    (tests/golden/c3_reference_digest.json, 4,999,950,000 bytes), their concatenation to its whole-payload digest,
    and the fused statistics equal its ComputeStats."""
    from concurrent.futures import ThreadPoolExecutor
    gold = json.loads((GOLDEN / "c3_reference_digest.json").read_text())
    ids, lens, sch = synth.config_store("C3")
    assert synth.store_digest(ids, lens) == gold["store_digest"] and list(sch) == gold["scheme"]
    P = nw.num_edges(len(lens))
    assert P == gold["edges"]
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        bounds = [int(b) for b in ctx.equal_work_bounds(8)]
        assert bounds == gold["shard_bounds"]
        host = torch.empty(P, dtype=torch.int8).pin_memory()
        tot, mn, mx = 0, 127, -128
        for g in range(8):
            st = ctx.score_range_host(bounds[g], bounds[g + 1], host[bounds[g]: bounds[g + 1]])
            assert st[3] == bounds[g + 1] - bounds[g]
            tot, mn, mx = tot + st[0], min(mn, st[1]), max(mx, st[2])
    view = memoryview(host.numpy()).cast("B")

    def digest(rng):
        return hashlib.blake2b(view[rng[0]: rng[1]], digest_size=16).hexdigest()

    with ThreadPoolExecutor(9) as ex:          # hashlib releases the GIL
        got = list(ex.map(digest, [(bounds[g], bounds[g + 1]) for g in range(8)] + [(0, P)]))
    assert got[:8] == gold["shard_blake2b_128"]
    assert got[8] == gold["payload_blake2b_128"]
    assert (mn, mx, tot / P) == (gold["min"], gold["max"], gold["mean"])


def test_c3_two_independent_kernels_agree():
    """configs[2] at full size (4,999,950,000 pairs): the packed DPX kernel and the int32
    one-thread-per-pair kernel must produce the same histogram / sum / min / max, and the same
    bytes on a strided sample of slabs."""
    ids, lens, sch = synth.config_store("C3")
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        P = ctx.num_edges
        a = torch.empty(P, dtype=torch.int8, device="cuda")
        sa = ctx.score_range(0, P, a, want_hist=True, variant="packed")
        assert sa[3] == P
        ps = ctx.payload_stats(a)
        assert ps[:4] == sa[:4] and np.array_equal(ps[4], sa[4])
        slab = 250_000_000
        b = torch.empty(slab, dtype=torch.int8, device="cuda")
        tot = [0, 127, -128, 0]
        hist = np.zeros(256, dtype=np.int64)
        for s in range(0, P, slab):
            e = min(P, s + slab)
            sb = ctx.score_range(s, e, b, want_hist=True, variant="simple")
            assert torch.equal(a[s:e], b[: e - s]), s
            tot = [tot[0] + sb[0], min(tot[1], sb[1]), max(tot[2], sb[2]), tot[3] + sb[3]]
            hist += sb[4]
        assert tuple(tot) == sa[:4] and np.array_equal(hist, sa[4])


def _slab_pass(ctx, variant, slab_bytes, want_hist=True, lo=0, hi=None):
    """Score [lo, hi) slab by slab into one reused device buffer; returns merged statistics."""
    hi = ctx.num_edges if hi is None else hi
    buf = torch.empty(slab_bytes, dtype=torch.int8, device="cuda")
    tot = [0, 127, -128, 0]
    hist = np.zeros(256, dtype=np.int64)
    for s in range(lo, hi, slab_bytes):
        e = min(hi, s + slab_bytes)
        st = ctx.score_range(s, e, buf, want_hist=want_hist, variant=variant)
        tot = [tot[0] + st[0], min(tot[1], st[1]), max(tot[2], st[2]), tot[3] + st[3]]
        if want_hist:
            hist += st[4]
    return tuple(tot), hist


# (the full-scale C4 / C5 protocol lives in tests/test_gpu_fullscale.py)


def test_c3_size_independent_properties():
    """configs[2] at full size, properties that need no oracle:
    (1) symmetry -- reversing the word ORDER maps edge (r, c) to (n-1-c, n-1-r) with the two words swapped,
        and nw_score(a, b) == nw_score(b, a) (reference tests/test_aligner.py:161-170), so the two payloads
        are related by an index permutation;
    (2) bounds -- gap*(la+lb) <= score <= match*min(la, lb) for gap <= min(mismatch, 0)
        (reference tests/test_aligner.py:172-184)."""
    ids, lens, sch = synth.config_store("C3")
    n = len(lens)
    m, x, g = sch
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as fwd, \
            NwapContext(ids[::-1].copy(), lens[::-1].copy(), nw.ScoringScheme(*sch)) as rev:
        P = fwd.num_edges
        a = torch.empty(P, dtype=torch.int8, device="cuda")
        b = torch.empty(P, dtype=torch.int8, device="cuda")
        sa = fwd.score_range(0, P, a)
        sb = rev.score_range(0, P, b)
        assert sa[:4] == sb[:4]                         # same multiset of scores
        lens_t = torch.as_tensor(lens.astype(np.int64), device="cuda")
        gen = torch.Generator(device="cuda").manual_seed(7)
        for _ in range(4):
            idx = torch.randint(0, P, (20_000_000,), generator=gen, device="cuda", dtype=torch.int64)
            rows = torch.empty_like(idx)
            cols = torch.empty_like(idx)
            _native.check(_native.lib().nwap_rows_cols(n, idx.data_ptr(), idx.numel(), rows.data_ptr(), cols.data_ptr(),
                                                       torch.cuda.current_stream().cuda_stream))
            r2, c2 = n - 1 - cols, n - 1 - rows
            idx2 = r2 * (2 * n - r2 - 1) // 2 + (c2 - r2 - 1)
            sc = a[idx].to(torch.int64)
            assert torch.equal(a[idx], b[idx2])
            la, lb = lens_t[rows], lens_t[cols]
            assert bool((sc <= m * torch.minimum(la, lb)).all()) and bool((sc >= g * (la + lb)).all())
        del a, b


# ---- new surface: compaction, degree, index recovery ----------------------------------------

def test_compaction_and_degree(golden_cases):
    c = golden_cases["seed500"]
    n, P = 500, nw.num_edges(500)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        ctx.score_range(0, P, out)
        for thr, (s, e) in [(2, (0, P)), (0, (1234, 99_000)), (-3, (P - 5000, P)), (100, (0, P))]:
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx, sc = ctx.compact_range(out[s:e], s, e, thr, capacity=e - s, degree=degree)
            ridx, rsc, rdeg = orc.np_compact(c["payload"][s:e], s, n, thr)
            assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
            assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
        with pytest.raises(_native.CapacityError) as ei:
            ctx.compact_range(out, 0, P, 0, capacity=10)
        assert ei.value.count == int((c["payload"] >= 0).sum())


def test_compaction_thresholds_alignments_and_tiny_ranges(golden_cases):
    """The vectorised compaction scan: every threshold class (<= -128 keeps all, > 127 keeps none, both
    halves of the unsigned byte order), payload pointers at every offset mod 16, ranges from 1 byte to
    several blocks, and the normalised filter on the same slices (its (r, c) walk starts mid-vector)."""
    c = golden_cases["seed500"]
    n, P = 500, nw.num_edges(500)
    lens64 = c["lengths"].astype(np.int64)
    rng = np.random.default_rng(99)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        big = torch.empty(P + 64, dtype=torch.int8, device="cuda")
        for off in range(17):
            out = big[off: off + P]
            ctx.score_range(0, P, out)
            spans = [(0, 1), (0, 15), (3, 20), (P - 1, P), (0, P), (16384 - off, 16384 - off + 1)]
            spans += [tuple(sorted(rng.integers(0, P, size=2))) for _ in range(3)]
            for s, e in spans:
                s, e = int(s), int(e)
                if e <= s:
                    continue
                thr = int(rng.choice([-200, -128, -127, -20, -3, -1, 0, 1, 2, 5, 127, 128, 300]))
                degree = torch.zeros(n, dtype=torch.int32, device="cuda")
                idx, sc = ctx.compact_range(out[s:e], s, e, thr, capacity=e - s, degree=degree)
                ridx, rsc, rdeg = orc.np_compact(c["payload"][s:e], s, n, thr)
                assert np.array_equal(idx.cpu().numpy(), ridx), (off, s, e, thr)
                assert np.array_equal(sc.cpu().numpy(), rsc)
                assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
                lo, hi = sorted(float(x) for x in rng.uniform(-120, 60, size=2))
                idx2, sc2 = ctx.filter_normalized(out[s:e], s, e, lo, hi, capacity=e - s)
                k = np.arange(s, e, dtype=np.int64)
                rows = orc.np_rows_of(k, n)
                cols = orc.np_cols_of(k, n, rows)
                w = 100.0 * c["payload"][s:e].astype(np.float64) / np.maximum(lens64[rows], lens64[cols])
                keep = (w >= lo) & (w <= hi)
                assert np.array_equal(idx2.cpu().numpy(), k[keep]), (off, s, e, lo, hi)
                assert np.array_equal(sc2.cpu().numpy(), c["payload"][s:e][keep])


def test_c5_threshold_compaction_slab(golden_samples):
    """configs[4]: alternate scheme (2,-1,-3), keep score >= 4, on a slab of the 600k job."""
    ids, lens, sch = synth.config_store("C5")
    n = len(lens)
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        P = ctx.num_edges
        s, e = P // 3, P // 3 + 3_000_000
        out = torch.empty(e - s, dtype=torch.int8, device="cuda")
        ctx.score_range(s, e, out)
        ref, *_ = _oracle(ids, lens, nw.ScoringScheme(*sch), s, e, threads=8)
        assert np.array_equal(out.cpu().numpy(), ref)
        degree = torch.zeros(n, dtype=torch.int32, device="cuda")
        idx, sc = ctx.compact_range(out, s, e, synth.C5_THRESHOLD, capacity=e - s, degree=degree)
        ridx, rsc, rdeg = orc.np_compact(ref, s, n, synth.C5_THRESHOLD)
        assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
        assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)


def test_normalized_filter_and_histogram_match_reference(golden_cases):
    """graph.py:91-101 keep-mask and store.py:342-381 normalised histogram on
    the device, against vectors produced by the reference's own filter_view / histogram."""
    c = golden_cases["seed500"]
    g = np.load(GOLDEN / "consumers_seed500.npz")
    n, P = 500, nw.num_edges(500)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        ctx.score_range(0, P, out)
        hn = ctx.hist_normalized(out, 0, P).cpu().numpy()
        first = int(g["hist_norm_first"][0])
        ref = np.zeros(25501, dtype=np.int64)
        ref[first + 12800: first + 12800 + len(g["hist_norm_counts"])] = g["hist_norm_counts"]
        assert np.array_equal(hn, ref)
        for k in range(5):
            lo, hi = (float(x) for x in g[f"filter{k}_bounds"])
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx, sc = ctx.filter_normalized(out, 0, P, lo, hi, capacity=P, degree=degree)
            assert idx.numel() == int(g[f"filter{k}_count"][0])
            assert np.array_equal(degree.cpu().numpy().astype(np.int64), g[f"filter{k}_degree"])
            idx_h = idx.cpu().numpy()
            assert np.array_equal(sc.cpu().numpy(), c["payload"][idx_h])
            if f"filter{k}_edges" in g:
                rows = orc.np_rows_of(idx_h, n)
                cols = orc.np_cols_of(idx_h, n, rows)
                assert np.array_equal(np.stack([rows, cols], 1), g[f"filter{k}_edges"].astype(np.int64))
        # sub-range + accumulate: two halves give the same histogram; odd offsets exercise the (r, c) walk
        acc = ctx.hist_normalized(out[: 70_001], 0, 70_001)
        acc = ctx.hist_normalized(out[70_001:], 70_001, P, counts=acc)
        assert np.array_equal(acc.cpu().numpy(), ref)
        with pytest.raises(ValueError):
            ctx.filter_normalized(out, 0, P, 2.0, 1.0, capacity=10)


def test_normalized_consumers_on_c5_slab():
    """The same consumers at configs[4] scale on a 3 M-edge slab, against the numpy restatement."""
    ids, lens, sch = synth.config_store("C5")
    n = len(lens)
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        P = ctx.num_edges
        s, e = 2 * (P // 3) + 17, 2 * (P // 3) + 17 + 3_000_000
        out = torch.empty(e - s, dtype=torch.int8, device="cuda")
        ctx.score_range(s, e, out)
        payload = out.cpu().numpy()
        ridx, rsc, rdeg = orc.np_filter_normalized(payload, s, n, lens, 25.0, 80.0)
        degree = torch.zeros(n, dtype=torch.int32, device="cuda")
        idx, sc = ctx.filter_normalized(out, s, e, 25.0, 80.0, capacity=e - s, degree=degree)
        assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
        assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
        assert np.array_equal(ctx.hist_normalized(out, s, e).cpu().numpy(), orc.np_hist_normalized(payload, s, n, lens))


def test_device_index_recovery(golden_triangle):
    t = golden_triangle
    for n in (4, 300, 10 ** 5, 10 ** 6, 10 ** 7, 600_000):
        rows, cols = device_rows_cols(t[f"n{n}_idx"], n)
        assert np.array_equal(rows, t[f"n{n}_rows"]) and np.array_equal(cols, t[f"n{n}_cols"])
    # exhaustive bijection for small n (tests/test_acceptance.py:136-153)
    for n in (2, 3, 17, 129, 300):
        idx = np.arange(nw.num_edges(n), dtype=np.int64)
        rows, cols = device_rows_cols(idx, n)
        assert (rows < cols).all() and (cols <= n - 1).all()
        assert np.array_equal(rows * (2 * n - rows - 1) // 2 + (cols - rows - 1), idx)


def test_launch_counter_moves():
    before = _native.lib().nwap_launch_count()
    c_ids = np.ones((10, 3), dtype=np.uint8)
    with NwapContext(c_ids, np.full(10, 3, dtype=np.uint8), nw.ScoringScheme()) as ctx:
        ctx.score_range(0, 45, torch.empty(45, dtype=torch.int8, device="cuda"))
    assert _native.lib().nwap_launch_count() >= before + 2
