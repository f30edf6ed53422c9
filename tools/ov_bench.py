"""Sparse override scheme (a handful of overridden pairs) at 20,000 French-shaped words: sparse-override cell
(packed3 with corrections) vs the table-driven cell vs the generic kernel vs the same scheme without overrides."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
ids, lens = synth.french_shaped(n)
cells = synth.total_cells(lens)
P = nw.num_edges(n)
ov = {(0, 1): 0, (2, 5): 1, (3, 4): 0, (7, 9): -2, (10, 11): 0, (0, 6): 1}       # the 11 most frequent symbols: 59 % of all matrix rows
ov_rare = {(20, 21): 0, (25, 30): 1, (33, 34): 0, (22, 38): -2, (27, 28): 0, (20, 36): 1}   # symbols of rank 20+: 11 % of the rows
for name, scheme, variants in (("uniform", nw.ScoringScheme(1, -1, -2), ("packed3",)),
                               ("6 pairs, rare symbols", nw.ScoringScheme(1, -1, -2, overrides=ov_rare), ("packed3", "packed_tab")),
                               ("6 overridden pairs", nw.ScoringScheme(1, -1, -2, overrides=ov), ("packed3", "packed_tab") + (("simple",) if n <= 20000 else ()))):
    with NwapContext(ids, lens, scheme) as ctx:
        out = torch.empty(P, dtype=torch.int8, device="cuda")
        ref = None
        for v in variants:
            ctx.score_range(0, P, out, variant=v)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ctx.score_range(0, P, out, variant=v, sync=False); e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            h = out.cpu().numpy()
            if ref is None: ref = h
            print(f"{name:22s} {v:12s} {ms:9.3f} ms  {cells / ms / 1e6:8.0f} GCUPS   same bytes: {bool(np.array_equal(h, ref))}")
