"""configs[3] / configs[4] (600,000 words, 179,999,700,000 edges) on ONE B200: the bit-exactness protocol of
SURVEY 8(d).

* the reference's own chunk digests (tests/golden/fullscale_chunks.json: 256 evenly spaced 65,536-edge chunks,
  first / last, one chunk either side of every equal-work shard bound) on three kernels, with the kept list of
  the threshold compaction and the kept edges' (row, col) -- dense path and sparse-output path;
* byte equality with the C oracle on more than 1e9 pairs per config;
* the packed kernel against the independent one-thread-per-pair kernel, BYTES per window;
* the whole C5 job in ONE sparse-output call against the shard-by-shard dense path + nwap_compact_range;
* opt-in (NWAP_FULL=1): the independent kernel over the whole job.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext, device_rows_cols
from oracle import nw_oracle as orc
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _b2(*arrays):
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def chunks():
    return json.loads((GOLDEN / "fullscale_chunks.json").read_text())


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_fullscale_chunks_against_the_reference(cfg, chunks):
    g = chunks[cfg]
    ids, lens, sch = synth.config_store(cfg)
    n = len(lens)
    assert synth.store_digest(ids, lens) == g["store_digest"]
    thr = g["threshold"]
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        assert [int(b) for b in ctx.equal_work_bounds(8)] == g["equal_work_bounds_8"]
        buf = torch.empty(chunks["chunk"] + 16, dtype=torch.int8, device="cuda")
        for k, r in enumerate(g["chunks"]):
            s, e = r["start"], r["end"]
            variants = ("auto", "packed", "simple") if (k % 4 == 0 or not r["tag"].startswith("even256")) else ("auto",)
            for v in variants:
                out = buf[(k % 16): (k % 16) + e - s]
                st = ctx.score_range(s, e, out, variant=v)
                assert _b2(out.cpu().numpy()) == r["blake2b_128"], (cfg, r["tag"], v)
                assert st[:4] == (r["sum"], r["min"], r["max"], e - s)
            # threshold compaction: dense payload -> nwap_compact_range, and the fused sparse output
            degree = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx, sc = ctx.compact_range(out, s, e, thr, capacity=e - s, degree=degree)
            idx_h, sc_h = idx.cpu().numpy(), sc.cpu().numpy()
            assert idx_h.size == r["kept"] and _b2(idx_h, sc_h) == r["kept_blake2b_128"], (cfg, r["tag"])
            degree2 = torch.zeros(n, dtype=torch.int32, device="cuda")
            idx2, sc2, st2 = ctx.score_range_compact(s, e, threshold=thr, capacity=r["kept"], degree=degree2)
            assert torch.equal(idx2, idx) and torch.equal(sc2, sc) and torch.equal(degree2, degree)
            assert st2 == (r["sum"], r["min"], r["max"], e - s)
            if idx_h.size:
                rows, cols = device_rows_cols(idx_h, n)
                assert _b2(rows, cols) == r["kept_rc_blake2b_128"]
                deg = np.bincount(rows, minlength=n) + np.bincount(cols, minlength=n)
                assert np.array_equal(degree.cpu().numpy().astype(np.int64), deg)


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_fullscale_bytes_vs_oracle_on_1e9_pairs(cfg, chunks):
    """17 windows of 60 M pairs: evenly spaced, plus windows straddling every interior shard bound and the end
    of the payload (1.02e9 pairs per config), every byte against oracle/nw_oracle.c."""
    g = chunks[cfg]
    ids, lens, sch = synth.config_store(cfg)
    n = len(lens)
    P = g["num_edges"]
    win = 60_000_000
    starts = [k * (P // 9) + 12_345 for k in range(9)] + [b - win // 2 for b in g["equal_work_bounds_8"][1:8]] + [P - win]
    sim = orc.similarity_matrix(sch[0], sch[1], int(ids.max()) + 1)
    ids32, len32 = ids.astype(np.int32), lens.astype(np.int32)
    threads = len(os.sched_getaffinity(0))
    total = 0
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        out = torch.empty(win, dtype=torch.int8, device="cuda")
        for s in starts:
            e = min(P, s + win)
            st = ctx.score_range(s, e, out)
            ref, rsum, rmin, rmax = orc.c_score_range(ids32, len32, sim, sch[2], n, s, e, threads=threads)
            got = out[: e - s].cpu().numpy()
            assert np.array_equal(got, ref), (cfg, s)
            assert st[:4] == (rsum, rmin, rmax, e - s)
            total += e - s
    assert total >= 1_000_000_000


def _window_pass(ctx, variant, lo, hi, buf):
    st = ctx.score_range(lo, hi, buf, want_hist=True, variant=variant)
    return st


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_full_scale_600k_two_kernels_agree_bytewise(cfg):
    """The whole job on the packed kernel (count, histogram, sum self-consistent), and on every 16th 500 M-edge
    window the independent one-thread-per-pair kernel must produce the same BYTES (22 windows, 1.1e10 pairs)."""
    ids, lens, sch = synth.config_store(cfg)
    full = os.environ.get("NWAP_FULL") == "1"
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        P = ctx.num_edges
        assert P == 179_999_700_000
        win = 500_000_000
        a = torch.empty(win, dtype=torch.int8, device="cuda")
        b = torch.empty(win, dtype=torch.int8, device="cuda")
        tot = [0, 127, -128, 0]
        hist = np.zeros(256, dtype=np.int64)
        checked = 0
        for k, s in enumerate(range(0, P, win)):
            e = min(P, s + win)
            sa = ctx.score_range(s, e, a, want_hist=True, variant="auto")
            tot = [tot[0] + sa[0], min(tot[1], sa[1]), max(tot[2], sa[2]), tot[3] + sa[3]]
            hist += sa[4]
            if full or k % 16 == 3:
                sb = ctx.score_range(s, e, b, want_hist=True, variant="simple")
                assert torch.equal(a[: e - s], b[: e - s]), (cfg, s)
                assert sa[:4] == sb[:4] and np.array_equal(sa[4], sb[4])
                checked += e - s
        assert tot[3] == P == int(hist.sum())
        assert int((hist * (np.arange(256) - 128)).sum()) == tot[0]
        nz = np.flatnonzero(hist)
        assert (int(nz[0]) - 128, int(nz[-1]) - 128) == (tot[1], tot[2])
        assert checked >= 11_000_000_000


def test_c5_whole_job_in_one_sparse_call():
    """BASELINE configs[4] on ONE GPU in ONE call: 1.8e11 edges scored, kept edges (score >= 4) and degree
    counts out, no dense payload anywhere.  Checked against the dense route the 8-GPU job takes: each
    equal-work shard scored into a 22.5 GB buffer and compacted by nwap_compact_range."""
    ids, lens, sch = synth.config_store("C5")
    n = len(lens)
    thr = synth.C5_THRESHOLD
    with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
        P = ctx.num_edges
        degree = torch.zeros(n, dtype=torch.int32, device="cuda")
        idx, sc, st = ctx.score_range_compact(0, P, threshold=thr, capacity=8_000_000, degree=degree)
        assert st[3] == P
        assert bool((idx[1:] > idx[:-1]).all())
        assert int(degree.sum().item()) == 2 * idx.numel()
        bounds = ctx.equal_work_bounds(8)
        buf = torch.empty(int(max(bounds[g + 1] - bounds[g] for g in range(8))), dtype=torch.int8, device="cuda")
        degree2 = torch.zeros(n, dtype=torch.int32, device="cuda")
        pos = 0
        tot = [0, 127, -128, 0]
        for g in range(8):
            s, e = int(bounds[g]), int(bounds[g + 1])
            sg = ctx.score_range(s, e, buf)
            tot = [tot[0] + sg[0], min(tot[1], sg[1]), max(tot[2], sg[2]), tot[3] + sg[3]]
            gi, gs = ctx.compact_range(buf, s, e, thr, capacity=2_000_000, degree=degree2)
            k = gi.numel()
            assert torch.equal(idx[pos: pos + k], gi) and torch.equal(sc[pos: pos + k], gs), g
            pos += k
        assert pos == idx.numel()
        assert torch.equal(degree, degree2)
        assert tuple(tot) == st
