"""Small all-variant run used under compute-sanitizer (memcheck / racecheck)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext
from oracle import nw_oracle as orc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2300
ids, lens = synth.french_shaped(n)
P = nw.num_edges(n)
sim = orc.similarity_matrix(1, -1, int(ids.max()) + 1)
ref, rsum, rmin, rmax = orc.c_score_range(ids.astype(np.int32), lens.astype(np.int32), sim, -2, n, 0, P, threads=4)
with NwapContext(ids, lens, nw.ScoringScheme(1, -1, -2)) as ctx:
    for variant in ("packed", "packed3", "packed_sym", "simple"):
        out = torch.empty(P + 3, dtype=torch.int8, device="cuda")[3:]
        st = ctx.score_range(5, P - 7, out, want_hist=True, variant=variant)
        got = out[: P - 12].cpu().numpy()
        assert np.array_equal(got, ref[5:P - 7]), variant
        print(variant, "ok", st[:4])
    deg = torch.zeros(n, dtype=torch.int32, device="cuda")
    idx, sc = ctx.compact_range(out[: P - 12], 5, P - 7, 2, capacity=P, degree=deg)
    print("compact kept", idx.numel(), ctx.payload_stats(out[: P - 12])[:4])

# round 2 paths: sparse output (raw threshold and normalised bounds), override schemes (sparse-correction and
# table-driven cells), words of 33..64 symbols (wide build), normalised consumers
with NwapContext(ids, lens, nw.ScoringScheme(1, -1, -2)) as ctx:
    deg = torch.zeros(n, dtype=torch.int32, device="cuda")
    idx, sc, st = ctx.score_range_compact(5, P - 7, threshold=2, capacity=P, degree=deg)
    keep = np.flatnonzero(ref[5:P - 7] >= 2) + 5
    assert np.array_equal(idx.cpu().numpy(), keep) and np.array_equal(sc.cpu().numpy(), ref[keep]), "sparse output"
    print("sparse ok", idx.numel())
    out = torch.empty(P, dtype=torch.int8, device="cuda")
    ctx.score_range(0, P, out)
    fi, fs = ctx.filter_normalized(out, 0, P, 40.0, 100.0, capacity=P)
    h = ctx.hist_normalized(out, 0, P)
    assert int(h.sum()) == P
    print("normalised consumers ok", fi.numel())
ov = {(0, 1): 0, (2, 5): 1, (3, 4): 0, (0, 6): 1}
sch = nw.ScoringScheme(1, -1, -2, overrides=ov)
simo = orc.similarity_matrix(1, -1, int(ids.max()) + 1, ov)
refo, *_ = orc.c_score_range(ids.astype(np.int32), lens.astype(np.int32), simo, -2, n, 0, P, threads=4)
with NwapContext(ids, lens, sch) as ctx:
    for variant in ("packed3", "packed_tab"):
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        ctx.score_range(0, P, out, variant=variant)
        assert np.array_equal(out.cpu().numpy(), refo), variant
        print("override", variant, "ok")
rng = np.random.default_rng(3)
n2 = 700
lens2 = rng.integers(1, 13, size=n2).astype(np.uint8)
lens2[rng.choice(n2, 40, replace=False)] = rng.integers(33, 65, size=40)
ids2 = rng.integers(0, 30, size=(n2, 64)).astype(np.uint8)
P2 = nw.num_edges(n2)
sim2 = orc.similarity_matrix(1, -1, 30)
ref2, *_ = orc.c_score_range(ids2.astype(np.int32), lens2.astype(np.int32), sim2, -1, n2, 0, P2, threads=4)
with NwapContext(ids2, lens2, nw.ScoringScheme(1, -1, -1)) as ctx:
    out = torch.empty(P2, dtype=torch.int8, device="cuda")
    ctx.score_range(0, P2, out)
    assert np.array_equal(out.cpu().numpy(), ref2), "wide"
    print("wide ok")
# override scheme over the same long-word vocabulary (wide build of the table-driven cell) and its sparse output
ov2 = {(0, 1): 0, (2, 5): 1, (3, 4): 0, (0, 6): 1}
sch2 = nw.ScoringScheme(1, -1, -1, overrides=ov2)
sim2o = orc.similarity_matrix(1, -1, 30, ov2)
ref2o, *_ = orc.c_score_range(ids2.astype(np.int32), lens2.astype(np.int32), sim2o, -1, n2, 0, P2, threads=4)
with NwapContext(ids2, lens2, sch2) as ctx:
    out = torch.empty(P2, dtype=torch.int8, device="cuda")
    ctx.score_range(0, P2, out)
    assert np.array_equal(out.cpu().numpy(), ref2o), "override wide"
    deg = torch.zeros(n2, dtype=torch.int32, device="cuda")
    idx, sc, st = ctx.score_range_compact(0, P2, threshold=1, capacity=P2, degree=deg)
    keep = np.flatnonzero(ref2o >= 1)
    assert np.array_equal(idx.cpu().numpy(), keep) and np.array_equal(sc.cpu().numpy(), ref2o[keep]), "override wide sparse"
    print("override wide ok", idx.numel())
with NwapContext(ids, lens, sch) as ctx:
    deg = torch.zeros(n, dtype=torch.int32, device="cuda")
    idx, sc, st = ctx.score_range_compact(5, P - 7, threshold=2, capacity=P, degree=deg)
    keep = np.flatnonzero(refo[5:P - 7] >= 2) + 5
    assert np.array_equal(idx.cpu().numpy(), keep) and np.array_equal(sc.cpu().numpy(), refo[keep]), "override sparse output"
    print("override sparse ok", idx.numel())
