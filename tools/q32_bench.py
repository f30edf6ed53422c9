"""Vocabularies whose longest word has 25..32 symbols: the 32-wide instantiation (no fast2 family, spills) against the
wide build (24-wide bodies + block-wise path for the long chunks).  NWAP_LIB selects the build (tools/ab.sh style)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext

base_ids, base_lens = synth.french_shaped(100_000)
for name, scheme in (("uniform 1/-1/-2", nw.ScoringScheme(1, -1, -2)),
                     ("6 overrides", nw.ScoringScheme(1, -1, -2, overrides={(0, 1): 0, (2, 5): 1, (3, 4): 0, (7, 9): -2, (10, 11): 0, (0, 6): 1}))):
    for frac in (0.001, 0.01):
        rng = np.random.default_rng(11)
        lens2 = base_lens.copy()
        q = 32
        ids2 = np.zeros((len(lens2), q), dtype=np.uint8)
        ids2[:, : base_ids.shape[1]] = base_ids
        pick = rng.choice(len(lens2), size=int(frac * len(lens2)), replace=False)
        lens2[pick] = rng.integers(25, 33, size=pick.size)
        ids2[pick] = rng.integers(0, 40, size=(pick.size, q))
        cells = synth.total_cells(lens2)
        with NwapContext(ids2, lens2, scheme) as ctx:
            P = ctx.num_edges
            buf = torch.empty(P, dtype=torch.int8, device="cuda")
            ts = []
            for rep in range(4):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); ctx.score_range(0, P, buf, sync=False); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            t = float(np.median(ts[1:]))
            print(f"{name:16s} {frac * 100:4.1f} % words of 25..32 symbols: {t:8.3f} ms  {cells / t / 1e6:8.0f} GCUPS  checksum {int(buf[::997].sum().item())}")
            del buf
