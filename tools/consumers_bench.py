"""HBM-bound consumers of the dense payload on one 22.5 GB shard of configs[4] (600k words, shard 0 of 8):
threshold compaction + degree (k_compact_count / k_compact_scan / k_compact_write), raw statistics +
histogram (k_payload_stats), normalised filter and normalised histogram.  CUDA-event times, GB/s of the
algorithmic traffic (1 byte read per edge per pass that reads it).  Run under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` for the per-kernel view."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext

ids, lens, sch = synth.config_store("C5")
n = len(lens)
res = {}
with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
    b = ctx.equal_work_bounds(8)
    s, e = int(b[0]), int(b[1])
    out = torch.empty(e - s, dtype=torch.int8, device="cuda")
    ctx.score_range(s, e, out)
    degree = torch.zeros(n, dtype=torch.int32, device="cuda")

    def timed(name, fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[name] = {"ms": best, "GBps_per_pass": (e - s) / best / 1e6}
        print(f"{name:28s} {best:8.3f} ms   {(e - s) / best / 1e6:8.1f} GB/s of payload", flush=True)
        return r

    step = 1 << 31
    def compact():
        k = 0
        for a in range(s, e, step):
            bb = min(e, a + step)
            idx, sc_ = ctx.compact_range(out[a - s: bb - s], a, bb, synth.C5_THRESHOLD, capacity=1 << 24, degree=degree)
            k += idx.numel()
        return k
    res["kept"] = timed("threshold compaction+degree", compact)
    timed("payload_stats (hist 256)", lambda: ctx.payload_stats(out, e - s))
    def nfilter():
        k = 0
        for a in range(s, e, step):
            bb = min(e, a + step)
            idx, sc_ = ctx.filter_normalized(out[a - s: bb - s], a, bb, 40.0, 100.0, capacity=1 << 26)
            k += idx.numel()
        return k
    res["kept_normalized_40_100"] = timed("normalised filter [40,100]", nfilter)
    def nhist():
        acc = None
        for a in range(s, e, step):
            bb = min(e, a + step)
            acc = ctx.hist_normalized(out[a - s: bb - s], a, bb, counts=acc)
        return acc
    timed("normalised histogram", nhist)
res["pairs"] = e - s
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/consumers_bench.json").write_text(json.dumps({k: (v if not torch.is_tensor(v) else None) for k, v in res.items()}, indent=1))
