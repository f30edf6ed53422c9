"""The two normalised consumers alone on one 2 GiB slice of a configs[4] shard (for ncu --set full captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext

ids, lens, sch = synth.config_store("C5")
with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
    b = ctx.equal_work_bounds(8)
    s = int(b[0]); e = s + (1 << 31)
    out = torch.empty(e - s, dtype=torch.int8, device="cuda")
    ctx.score_range(s, e, out)
    for _ in range(2):
        idx, sc_ = ctx.filter_normalized(out, s, e, 40.0, 100.0, capacity=1 << 26)
        acc = ctx.hist_normalized(out, s, e)
    torch.cuda.synchronize()
    print("kept", idx.numel(), "hist total", int(acc.sum()))
