"""Round-2 kernels through the C ABI:

* sparse-output mode (nwap_score_range_compact / _filter_normalized): the threshold compaction fused into the
  tile kernel's writer must give exactly what nwap_compact_range / nwap_filter_normalized give over the
  dense payload -- which in turn are pinned to numpy over reference-produced payloads;
* words of 25..64 symbols (the int8 preflight admits 64 for gap -1, reference engine.py:83-90) on the packed
  kernel's block-wise path: golden `long40` (reference-generated), random long vocabularies vs the oracle.
"""
import numpy as np
import pytest

import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import _native, synth
from paper_2509_01654_b200.engine import NwapContext
from oracle import nw_oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _scheme(case):
    m, x, g = case["scheme"]
    return nw.ScoringScheme(m, x, g, overrides={(a, b): v for a, b, v in case.get("overrides", [])})


def _oracle(ids, lens, scheme, start, end, threads=8):
    sim = orc.similarity_matrix(scheme.match, scheme.mismatch, int(ids.max()) + 1, dict(scheme.overrides))
    return orc.c_score_range(ids.astype(np.int32), lens.astype(np.int32), sim, scheme.gap, len(lens), start, end,
                             threads=threads)


# ---------------------------------------------------------------------------------- sparse output

def test_sparse_output_equals_compaction_of_the_dense_payload(golden_cases):
    """Every threshold class, ranges that start and end mid-row, dense payload requested or not, degree."""
    c = golden_cases["seed500"]
    n, P = 500, nw.num_edges(500)
    ref = c["payload"]
    rng = np.random.default_rng(5)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        spans = [(0, P), (0, 1), (P - 1, P), (1234, 99_000), (P - 5000, P), (498, 500), (0, 499)]
        spans += [tuple(sorted(int(x) for x in rng.integers(0, P, size=2))) for _ in range(12)]
        for k, (s, e) in enumerate(spans):
            if e <= s:
                continue
            thr = int(rng.choice([-200, -128, -127, -20, -3, -1, 0, 1, 2, 5, 127, 128, 300]))
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            dense = torch.full((e - s + 32,), 0x55, dtype=torch.int8, device="cuda") if k % 2 else None
            out = dense[7: 7 + e - s] if dense is not None else None
            idx, sc, st = ctx.score_range_compact(s, e, threshold=thr, capacity=e - s, out=out, degree=degree)
            ridx, rsc, rdeg = orc.np_compact(ref[s:e], s, n, thr)
            assert np.array_equal(idx.cpu().numpy(), ridx), (s, e, thr)
            assert np.array_equal(sc.cpu().numpy(), rsc)
            assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
            sub = ref[s:e].astype(np.int64)
            assert st == (int(sub.sum()), int(sub.min()), int(sub.max()), e - s)
            if dense is not None:
                host = dense.cpu().numpy()
                assert np.array_equal(host[7: 7 + e - s], ref[s:e])
                assert (host[:7] == 0x55).all() and (host[7 + e - s:] == 0x55).all()
        with pytest.raises(_native.CapacityError) as ei:
            ctx.score_range_compact(0, P, threshold=0, capacity=10)
        assert ei.value.count == int((ref >= 0).sum())
        with pytest.raises(ValueError):
            ctx.score_range_compact(0, P, capacity=10)


def test_sparse_output_normalized_filter_matches_reference_vectors(golden_cases):
    """graph.py:91-101 keep-mask evaluated where the scores are produced, against the reference's own
    filter_view results (tests/golden/consumers_seed500.npz) and numpy on sub-ranges."""
    from conftest import GOLDEN
    c = golden_cases["seed500"]
    g = np.load(GOLDEN / "consumers_seed500.npz")
    n, P = 500, nw.num_edges(500)
    lens64 = c["lengths"].astype(np.int64)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        for k in range(5):
            lo, hi = (float(x) for x in g[f"filter{k}_bounds"])
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx, sc, _ = ctx.score_range_compact(0, P, normalized=(lo, hi), capacity=P, degree=degree)
            assert idx.numel() == int(g[f"filter{k}_count"][0])
            assert np.array_equal(degree.cpu().numpy().astype(np.int64), g[f"filter{k}_degree"])
            idx_h = idx.cpu().numpy()
            assert np.all(np.diff(idx_h) > 0)
            assert np.array_equal(sc.cpu().numpy(), c["payload"][idx_h])
        rng = np.random.default_rng(17)
        for _ in range(10):
            s, e = sorted(int(x) for x in rng.integers(0, P, size=2))
            if e <= s:
                continue
            lo, hi = sorted(float(x) for x in rng.uniform(-120, 60, size=2))
            idx, sc, _ = ctx.score_range_compact(s, e, normalized=(lo, hi), capacity=e - s)
            k = np.arange(s, e, dtype=np.int64)
            rows = orc.np_rows_of(k, n)
            cols = orc.np_cols_of(k, n, rows)
            w = 100.0 * c["payload"][s:e].astype(np.float64) / np.maximum(lens64[rows], lens64[cols])
            keep = (w >= lo) & (w <= hi)
            assert np.array_equal(idx.cpu().numpy(), k[keep]), (s, e, lo, hi)
            assert np.array_equal(sc.cpu().numpy(), c["payload"][s:e][keep])


def test_sparse_output_c2_many_kept_edges():
    """20,000 words, threshold 0 keeps ~3 % of 2e8 edges (several million keys through the radix sort, five
    passes); identical to the dense path + nwap_compact_range, and a second call reuses the scratch."""
    ids, lens, sch = synth.config_store("C2")
    n = len(lens)
    scheme = nw.ScoringScheme(*sch)
    with NwapContext(ids, lens, scheme) as ctx:
        P = ctx.num_edges
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        st_dense = ctx.score_range(0, P, out)
        for thr in (0, 3):
            kept = int((out >= thr).sum().item())
            d1 = torch.zeros(n, dtype=torch.int32, device="cuda")
            d2 = torch.zeros(n, dtype=torch.int32, device="cuda")
            ridx, rsc = ctx.compact_range(out, 0, P, thr, capacity=kept, degree=d1)
            idx, sc, st = ctx.score_range_compact(0, P, threshold=thr, capacity=kept + 5, degree=d2)
            assert idx.numel() == kept
            assert torch.equal(idx, ridx) and torch.equal(sc, rsc) and torch.equal(d1, d2)
            assert st == st_dense[:4]


def test_sparse_output_c5_slab_and_shard_boundaries():
    """configs[4] (scheme 2/-1/-3, keep >= 4): a slab and the neighbourhood of two equal-work shard bounds of
    the 600k job, sparse output vs the oracle + numpy compaction."""
    ids, lens, sch = synth.config_store("C5")
    n = len(lens)
    scheme = nw.ScoringScheme(*sch)
    with NwapContext(ids, lens, scheme) as ctx:
        P = ctx.num_edges
        bounds = ctx.equal_work_bounds(8)
        for s, e in [(P // 3, P // 3 + 3_000_000), (int(bounds[3]) - 700_000, int(bounds[3]) + 700_000),
                     (int(bounds[7]) - 65_536, int(bounds[7]) + 65_536), (P - 2_000_000, P)]:
            ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, s, e)
            ridx, rsc, rdeg = orc.np_compact(ref, s, n, synth.C5_THRESHOLD)
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx, sc, st = ctx.score_range_compact(s, e, threshold=synth.C5_THRESHOLD, capacity=len(ridx) + 1, degree=degree)
            assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
            assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
            assert st == (rsum, rmin, rmax, e - s)


# ---------------------------------------------------------------------------------- long words

def test_long40_golden_runs_on_the_packed_kernel(golden_cases):
    """Reference-generated case with words of 20..40 symbols, scheme (1,-1,-1): `auto` must stay on the packed
    tile kernel (the launch is k_score_tiles, not k_score_simple) and reproduce the reference's bytes."""
    c = golden_cases["long40"]
    n = len(c["lengths"])
    P = nw.num_edges(n)
    with NwapContext(c["ids"], c["lengths"], _scheme(c)) as ctx:
        for variant in ("auto", "packed3", "simple"):
            out = torch.empty(P, dtype=torch.int8, device="cuda")
            st = ctx.score_range(0, P, out, variant=variant)
            assert np.array_equal(out.cpu().numpy(), c["payload"]), variant
            assert st[:4] == (int(c["payload"].astype(np.int64).sum()), int(c["payload"].min()), int(c["payload"].max()), P)
        with pytest.raises(ValueError):
            ctx.score_range(0, P, out, variant="packed")      # the 2-IMAD A/B build stays at 32 symbols


@pytest.mark.parametrize("qmax,gap", [(25, -2), (28, -2), (32, -2), (33, -1), (48, -1), (64, -1), (40, 0), (63, 1)])
def test_long_words_block_path_vs_oracle(qmax, gap):
    """Random vocabularies mixing short words with words of up to 64 symbols: all bytes + statistics vs the
    oracle, sub-ranges with misaligned outputs, and the sparse output on the wide build (which uniform schemes take
    from a longest word of 25 symbols on)."""
    rng = np.random.default_rng(1000 + qmax)
    n = 6000
    lens = np.clip(np.rint(rng.normal(8.5, 2.8, size=n)), 1, 24).astype(np.uint8)
    long_ix = rng.choice(n, size=n // 20, replace=False)
    lens[long_ix] = rng.integers(25, qmax + 1, size=long_ix.size)
    lens[rng.integers(0, n)] = qmax
    ids = rng.integers(0, 12, size=(n, qmax)).astype(np.uint8)
    match = 1 if gap < 0 else 0
    scheme = nw.ScoringScheme(match, -1, gap)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P)
    with NwapContext(ids, lens, scheme) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        st = ctx.score_range(0, P, out)
        got = out.cpu().numpy()
        bad = np.flatnonzero(got != ref)
        assert bad.size == 0, (bad[:5], got[bad[:5]], ref[bad[:5]])
        assert st[:4] == (rsum, rmin, rmax, P)
        for s, e, off in [(5, 77, 3), (P // 2 + 1, P // 2 + 100_001, 9), (P - 40_000, P, 15)]:
            buf = torch.full((e - s + 48,), 0x55, dtype=torch.int8, device="cuda")
            ctx.score_range(s, e, buf[off:])
            host = buf.cpu().numpy()
            assert np.array_equal(host[off: off + e - s], ref[s:e])
            assert (host[:off] == 0x55).all() and (host[off + e - s:] == 0x55).all()
        thr = int(np.percentile(ref, 99.9))
        ridx, rsc, rdeg = orc.np_compact(ref, 0, n, thr)
        degree = torch.zeros(n, dtype=torch.int32, device="cuda")
        idx, sc, st2 = ctx.score_range_compact(0, P, threshold=thr, capacity=len(ridx), degree=degree)
        assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
        assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
        assert st2 == (rsum, rmin, rmax, P)


def test_all_words_at_the_64_symbol_limit():
    """Every word 64 symbols, scheme (1,-1,-1): the extreme of the preflight (2*64*1 = 128)."""
    rng = np.random.default_rng(64)
    n = 700
    lens = np.full(n, 64, dtype=np.uint8)
    ids = rng.integers(0, 4, size=(n, 64)).astype(np.uint8)
    ids[: n // 2] = ids[0]                    # identical words: score 64 > ... must stay inside int8 (64 <= 127)
    scheme = nw.ScoringScheme(1, -1, -1)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P)
    with NwapContext(ids, lens, scheme) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        st = ctx.score_range(0, P, out)
        assert np.array_equal(out.cpu().numpy(), ref)
        assert st[:4] == (rsum, rmin, rmax, P)


# ------------------------------------------------------------- override schemes: long words, sparse output

def _override_scheme(rng, K, q, gap, dense):
    """A random override scheme the int8 preflight admits for words of up to q symbols (engine.py:72-96)."""
    lim = 127 // q
    if dense:
        lo_s, hi_s = -min(2, 128 // q), min(2, lim)
        ov = {(a, b): int(rng.integers(lo_s, hi_s + 1)) for a in range(K) for b in range(a, K)}
        return nw.ScoringScheme(ov[(0, 0)], ov[(0, 1)], gap, overrides=ov)
    m, x = min(1, lim), -1
    ov = {}
    for _ in range(6):
        a_, b_ = int(rng.integers(0, K)), int(rng.integers(0, K))
        ov[(min(a_, b_), max(a_, b_))] = int(rng.integers(-min(2, 128 // q), min(2, lim) + 1))
    return nw.ScoringScheme(m, x, gap, overrides=ov)


@pytest.mark.parametrize("qmax,K,dense", [(33, 12, False), (48, 40, True), (64, 40, False), (64, 7, True)])
def test_override_scheme_with_long_words_stays_on_the_packed_kernel(qmax, K, dense):
    """Override schemes over vocabularies with words of 33..64 symbols ran the generic one-thread-per-pair kernel
    (0.56 TCUPS); now `auto` takes the wide build of the table-driven cell (block-wise path for the long chunks).
    All bytes + statistics vs the oracle and vs the generic kernel, misaligned sub-ranges, sparse output."""
    rng = np.random.default_rng(7000 + qmax + K)
    n = 5000
    lens = np.clip(np.rint(rng.normal(8.5, 2.8, size=n)), 1, 24).astype(np.uint8)
    long_ix = rng.choice(n, size=n // 25, replace=False)
    lens[long_ix] = rng.integers(25, qmax + 1, size=long_ix.size)
    lens[rng.integers(0, n)] = qmax
    ids = rng.integers(0, K, size=(n, qmax)).astype(np.uint8)
    scheme = _override_scheme(rng, K, qmax, -1, dense)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P)
    with NwapContext(ids, lens, scheme) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        for variant in ("auto", "packed_tab"):
            out.fill_(0x55)
            st = ctx.score_range(0, P, out, variant=variant)
            got = out.cpu().numpy()
            bad = np.flatnonzero(got != ref)
            assert bad.size == 0, (variant, bad[:5], got[bad[:5]], ref[bad[:5]])
            assert st[:4] == (rsum, rmin, rmax, P)
        s, e = P // 3 + 7, P // 3 + 7 + 300_001
        ctx.score_range(s, e, out[5:], variant="simple")
        assert np.array_equal(out[5: 5 + e - s].cpu().numpy(), ref[s:e])
        for s, e, off in [(5, 77, 3), (P // 2 + 1, P // 2 + 100_001, 9), (P - 40_000, P, 15)]:
            buf = torch.full((e - s + 48,), 0x55, dtype=torch.int8, device="cuda")
            ctx.score_range(s, e, buf[off:])
            host = buf.cpu().numpy()
            assert np.array_equal(host[off: off + e - s], ref[s:e])
            assert (host[:off] == 0x55).all() and (host[off + e - s:] == 0x55).all()
        thr = int(np.percentile(ref, 99.9))
        ridx, rsc, rdeg = orc.np_compact(ref, 0, n, thr)
        degree = torch.zeros(n, dtype=torch.int32, device="cuda")
        idx, sc, st2 = ctx.score_range_compact(0, P, threshold=thr, capacity=len(ridx), degree=degree)
        assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
        assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
        assert st2 == (rsum, rmin, rmax, P)


@pytest.mark.parametrize("K,q,dense", [(40, 24, False), (40, 16, True), (128, 12, True), (9, 32, False)])
def test_sparse_output_of_an_override_scheme(K, q, dense):
    """The sparse-output mode of the edge writer on the table-driven kernel: kept list, degree and statistics equal
    the threshold compaction of the dense payload (numpy model over the oracle's bytes), with and without the dense
    payload written alongside."""
    rng = np.random.default_rng(9000 + K + q)
    n = 4000
    lens = rng.integers(1, q + 1, size=n).astype(np.uint8)
    lens[0] = q
    ids = rng.integers(0, K, size=(n, q)).astype(np.uint8)
    scheme = _override_scheme(rng, K, q, -2 if q <= 24 else -1, dense)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P)
    with NwapContext(ids, lens, scheme) as ctx:
        for thr in (int(np.percentile(ref, 99.5)), int(ref.max())):
            ridx, rsc, rdeg = orc.np_compact(ref, 0, n, thr)
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx, sc, st = ctx.score_range_compact(0, P, threshold=thr, capacity=len(ridx) + 5, degree=degree)
            assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
            assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
            assert st == (rsum, rmin, rmax, P)
        s, e = P // 5 + 3, P // 5 + 3 + 1_000_001
        thr = int(np.percentile(ref[s:e], 99.0))
        ridx, rsc, _ = orc.np_compact(ref[s:e], s, n, thr)
        dense_out = torch.full((e - s,), 0x55, dtype=torch.int8, device="cuda")
        idx, sc, _ = ctx.score_range_compact(s, e, threshold=thr, capacity=len(ridx), out=dense_out)
        assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
        assert np.array_equal(dense_out.cpu().numpy(), ref[s:e])


@pytest.mark.parametrize("scheme,overrides", [((1, -1, 0), None), ((1, 0, 0), None), ((1, -1, 0), {(0, 1): 0, (2, 3): 1})])
def test_words_over_64_symbols_fall_back_to_the_generic_kernel(scheme, overrides):
    """With gap 0 the int8 preflight admits words of up to 127 symbols (engine.py:83-90: 2*q*gap drops out).  The
    packed kernel stops at 64; `auto` then runs the generic one-thread-per-pair kernel -- same bytes as the oracle,
    and the packed variants refuse with the reference-facing error."""
    rng = np.random.default_rng(127)
    n, qmax, K = 900, 127, 9
    lens = np.clip(np.rint(rng.normal(8.5, 2.8, size=n)), 1, 24).astype(np.uint8)
    lens[rng.choice(n, size=30, replace=False)] = rng.integers(65, qmax + 1, size=30)
    lens[0] = qmax
    ids = rng.integers(0, K, size=(n, qmax)).astype(np.uint8)
    sch = nw.ScoringScheme(*scheme, overrides=overrides or {})
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, sch, 0, P)
    with NwapContext(ids, lens, sch) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        st = ctx.score_range(0, P, out)
        assert np.array_equal(out.cpu().numpy(), ref)
        assert st[:4] == (rsum, rmin, rmax, P)
        with pytest.raises(ValueError):
            ctx.score_range(0, P, out, variant="packed_tab" if overrides else "packed3")


def test_vocabulary_made_of_long_words_keeps_the_32_wide_build():
    """More than 40 % of the symbols in words of 25..32 symbols: `auto` keeps the 32-wide instantiation (every chunk
    would go block-wise on the wide build).  Bytes, statistics and the sparse output against the oracle."""
    rng = np.random.default_rng(3232)
    n, qmax = 3000, 32
    lens = rng.integers(18, qmax + 1, size=n).astype(np.uint8)
    lens[0] = qmax
    ids = rng.integers(0, 30, size=(n, qmax)).astype(np.uint8)
    scheme = nw.ScoringScheme(1, -1, -2)
    P = nw.num_edges(n)
    ref, rsum, rmin, rmax = _oracle(ids, lens, scheme, 0, P)
    with NwapContext(ids, lens, scheme) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        for variant in ("auto", "packed3", "packed", "simple"):
            out.fill_(0x55)
            st = ctx.score_range(0, P, out, variant=variant)
            assert np.array_equal(out.cpu().numpy(), ref), variant
            assert st[:4] == (rsum, rmin, rmax, P)
        thr = int(np.percentile(ref, 99.9))
        ridx, rsc, rdeg = orc.np_compact(ref, 0, n, thr)
        degree = torch.zeros(n, dtype=torch.int32, device="cuda")
        idx, sc, st2 = ctx.score_range_compact(0, P, threshold=thr, capacity=len(ridx), degree=degree)
        assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(sc.cpu().numpy(), rsc)
        assert np.array_equal(degree.cpu().numpy().astype(np.int64), rdeg)
        assert st2 == (rsum, rmin, rmax, P)
