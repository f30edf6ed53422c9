"""Where the end-to-end (host buffer) step spends its time: context create, scoring into pinned
host memory, destroy.  Diagnostic for bench.py's e2e figure."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
ids, lens = synth.french_shaped(n)
sch = nw.ScoringScheme(1, -1, -2)
P = nw.num_edges(n)
host = torch.empty(P, dtype=torch.int8).pin_memory()
torch.cuda.synchronize()
for rep in range(4):
    t0 = time.perf_counter()
    ctx = NwapContext(ids, lens, sch, device=0)
    t1 = time.perf_counter()
    r = ctx.score_range_host(0, P, host)
    t2 = time.perf_counter()
    r = ctx.score_range_host(0, P, host)
    t3 = time.perf_counter()
    ctx.close()
    t4 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, score_host(first) {1e3*(t2-t1):.1f} ms, "
          f"score_host(again) {1e3*(t3-t2):.1f} ms, destroy {1e3*(t4-t3):.1f} ms")
d = torch.empty(1 << 30, dtype=torch.int8, device="cuda")
for nb in (1 << 30, 256 << 20, 64 << 20, 16 << 20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for k in range((1 << 30) // nb):
        host[k * nb:(k + 1) * nb].copy_(d[k * nb:(k + 1) * nb], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"D2H 1 GiB in {nb >> 20} MiB pieces: {(1 << 30) / dt / 1e9:.1f} GB/s")
