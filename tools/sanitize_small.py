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
