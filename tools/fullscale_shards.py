"""configs[3] / configs[4] at full size on ONE GPU, shard by shard: the 600,000-word job is cut into
the 8 equal-work contiguous shards an 8-GPU run would use; each shard (~22.5 GB of
int8 output, fits one B200) is scored here in turn into the same device buffer, timed with CUDA
events, and cross-checked (count, and sum/min/max/hist against the independent k_payload_stats pass).
C5 also runs the threshold compaction + degree counts on every shard.

The max over shards is what an 8-GPU run's kernel time would be (no data-path collective); the
sum is the whole job on one GPU.  Writes gpurun_out/fullscale_<cfg>.json.
"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth
from paper_2509_01654_b200.engine import NwapContext

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ids, lens, sch = synth.config_store(cfg)
n = len(lens)
cells_total = synth.total_cells(lens)
res = {"config": cfg, "words": n, "scheme": list(sch), "parts": parts, "shards": []}
with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
    P = ctx.num_edges
    bounds = ctx.equal_work_bounds(parts)
    out = torch.empty(int(np.diff(bounds).max()), dtype=torch.int8, device="cuda")
    degree = torch.zeros(n, dtype=torch.int32, device="cuda") if cfg == "C5" else None
    tot_sum = tot_cnt = 0
    hist = np.zeros(256, dtype=np.int64)
    kept_total = 0
    for g in range(parts):
        s, e = int(bounds[g]), int(bounds[g + 1])
        ctx.score_range(s, min(e, s + 1000), out)                        # warm
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        ctx.score_range(s, e, out, sync=False)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        st = ctx.read_stats()
        t0 = time.perf_counter()
        ps = ctx.payload_stats(out, e - s)
        ps_ms = 1e3 * (time.perf_counter() - t0)
        assert st[:4] == ps[:4] and st[3] == e - s, (g, st[:4], ps[:4])
        cells = ctx.cells_in_range(s, e)
        rec = {"shard": g, "start": s, "end": e, "pairs": e - s, "cells": cells, "kernel_ms": ms,
               "gcups": cells / ms / 1e6, "pairs_per_s": (e - s) / ms * 1e3,
               "sum": st[0], "min": st[1], "max": st[2], "payload_stats_ms": ps_ms}
        if cfg == "C5":
            t0 = time.perf_counter()
            kept = 0
            step = 1 << 31                                             # compaction call limit: 2^31 blocks of 4096 edges is far above this
            for a in range(s, e, step):
                b = min(e, a + step)
                cap = 1 << 26
                idx, sc = ctx.compact_range(out[a - s: b - s], a, b, synth.C5_THRESHOLD, capacity=cap, degree=degree)
                kept += idx.numel()
            torch.cuda.synchronize()
            rec["compaction_ms"] = 1e3 * (time.perf_counter() - t0)
            rec["kept"] = kept
            kept_total += kept
        tot_sum += st[0]; tot_cnt += st[3]; hist += ps[4]
        res["shards"].append(rec)
        print(json.dumps(rec), flush=True)
    assert tot_cnt == P
    k = np.array([r["kernel_ms"] for r in res["shards"]])
    res.update(pairs=P, cells=cells_total, sum=tot_sum, mean=tot_sum / P,
               min=min(r["min"] for r in res["shards"]), max=max(r["max"] for r in res["shards"]),
               kernel_ms_total=float(k.sum()), kernel_ms_max=float(k.max()), kernel_ms_mean=float(k.mean()),
               balance_max_over_mean=float(k.max() / k.mean()),
               one_gpu_gcups=cells_total / k.sum() / 1e6, one_gpu_pairs_per_s=P / k.sum() * 1e3,
               projected_8gpu_gcups=cells_total / k.max() / 1e6, projected_8gpu_pairs_per_s=P / k.max() * 1e3,
               hist_nonzero={int(i) - 128: int(v) for i, v in enumerate(hist) if v})
    if cfg == "C5":
        res["kept_total"] = kept_total
        res["degree_sum"] = int(degree.sum(dtype=torch.int64).item())
        assert res["degree_sum"] == 2 * kept_total
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/fullscale_{cfg}.json").write_text(json.dumps(res, indent=1))
print({k: v for k, v in res.items() if k not in ("shards", "hist_nonzero")})
