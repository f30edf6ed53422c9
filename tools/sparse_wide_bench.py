"""Round-2 measurements on one B200 (CUDA events around the calls, medians):
  (1) sparse-output mode vs dense scoring (+ nwap_compact_range) at C3-size and on a C5 shard;
  (2) the whole C5 job (600k words) in one sparse-output call;
  (3) 100,000-word vocabulary with 0.1 % / 1 % words of 33..48 symbols, scheme (1,-1,-1): wide build vs the all-short rate.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2509_01654_b200 as nw  # noqa: E402
from paper_2509_01654_b200 import synth  # noqa: E402
from paper_2509_01654_b200.engine import NwapContext  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), r


out = {}
# (1) C3-size: dense vs sparse-only vs sparse+dense
ids, lens, sch = synth.config_store("C3")
cells = synth.total_cells(lens)
with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
    P = ctx.num_edges
    buf = torch.empty(P, dtype=torch.int8, device="cuda")
    t_dense, _ = timed(lambda: ctx.score_range(0, P, buf))
    for thr in (-2, 2):
        kept = int((buf >= thr).sum().item())
        t_cmp, _ = timed(lambda: ctx.compact_range(buf, 0, P, thr, capacity=kept))
        t_sparse, r = timed(lambda: ctx.score_range_compact(0, P, threshold=thr, capacity=kept))
        t_both, _ = timed(lambda: ctx.score_range_compact(0, P, threshold=thr, capacity=kept, out=buf))
        out[f"C3_thr{thr}"] = {"kept": kept, "dense_ms": t_dense, "compact_range_ms": t_cmp, "sparse_only_ms": t_sparse,
                               "sparse_plus_dense_ms": t_both, "sparse_over_dense": t_sparse / t_dense,
                               "gcups_sparse": cells / t_sparse / 1e6}
        print(json.dumps({f"C3_thr{thr}": out[f"C3_thr{thr}"]}), flush=True)
    del buf

# (2) C5 whole job, one call
ids, lens, sch = synth.config_store("C5")
cells = synth.total_cells(lens)
n = len(lens)
with NwapContext(ids, lens, nw.ScoringScheme(*sch)) as ctx:
    P = ctx.num_edges
    degree = torch.zeros(n, dtype=torch.int32, device="cuda")
    t, r = timed(lambda: ctx.score_range_compact(0, P, threshold=synth.C5_THRESHOLD, capacity=8_000_000, degree=degree), reps=3, warm=1)
    out["C5_one_call"] = {"ms": t, "kept": int(r[0].numel()), "gcups": cells / t / 1e6, "pairs_per_s": P / t * 1e3,
                          "stats": list(r[2])}
    print(json.dumps({"C5_one_call": out["C5_one_call"]}), flush=True)
    # scoring alone on the same job: 8 shards dense
    bounds = ctx.equal_work_bounds(8)
    buf = torch.empty(int(max(bounds[g + 1] - bounds[g] for g in range(8))), dtype=torch.int8, device="cuda")
    t8, _ = timed(lambda: [ctx.score_range(int(bounds[g]), int(bounds[g + 1]), buf, sync=False) for g in range(8)], reps=3, warm=1)
    out["C5_dense_8_shards_ms"] = t8
    out["C5_sparse_over_dense"] = t / t8
    print(json.dumps({"C5_dense_8_shards_ms": t8, "ratio": t / t8}), flush=True)
    del buf

# (3) long-word tail, scheme (1,-1,-1)
base_ids, base_lens = synth.french_shaped(100_000)
scheme = nw.ScoringScheme(1, -1, -1)
for frac in (0.0, 0.001, 0.01):
    rng = np.random.default_rng(7)
    lens2 = base_lens.copy()
    q = 48 if frac else int(base_lens.max())
    ids2 = np.zeros((len(lens2), q), dtype=np.uint8)
    ids2[:, : base_ids.shape[1]] = base_ids
    if frac:
        pick = rng.choice(len(lens2), size=int(frac * len(lens2)), replace=False)
        lens2[pick] = rng.integers(33, 49, size=pick.size)
        ids2[pick] = rng.integers(0, 40, size=(pick.size, q))
    cells = synth.total_cells(lens2)
    with NwapContext(ids2, lens2, scheme) as ctx:
        P = ctx.num_edges
        buf = torch.empty(P, dtype=torch.int8, device="cuda")
        t, _ = timed(lambda: ctx.score_range(0, P, buf, sync=False))
        out[f"long_tail_{frac}"] = {"ms": t, "gcups": cells / t / 1e6, "pairs_per_s": P / t * 1e3, "qmax": int(lens2.max())}
        print(json.dumps({f"long_tail_{frac}": out[f"long_tail_{frac}"]}), flush=True)
        del buf
# (4) the same with an OVERRIDE scheme (table-driven cell): long-word tail on its wide build, and its sparse output
ov = {(0, 1): 0, (2, 5): 1, (3, 4): 0, (7, 9): -1, (10, 11): 0, (0, 6): 1}
scheme_ov = nw.ScoringScheme(1, -1, -1, overrides=ov)
for frac in (0.0, 0.001, 0.01):
    rng = np.random.default_rng(7)
    lens2 = base_lens.copy()
    q = 48 if frac else int(base_lens.max())
    ids2 = np.zeros((len(lens2), q), dtype=np.uint8)
    ids2[:, : base_ids.shape[1]] = base_ids
    if frac:
        pick = rng.choice(len(lens2), size=int(frac * len(lens2)), replace=False)
        lens2[pick] = rng.integers(33, 49, size=pick.size)
        ids2[pick] = rng.integers(0, 40, size=(pick.size, q))
    cells = synth.total_cells(lens2)
    with NwapContext(ids2, lens2, scheme_ov) as ctx:
        P = ctx.num_edges
        buf = torch.empty(P, dtype=torch.int8, device="cuda")
        t, _ = timed(lambda: ctx.score_range(0, P, buf, sync=False))
        rec = {"ms": t, "gcups": cells / t / 1e6, "qmax": int(lens2.max())}
        if not frac:
            thr = 2
            kept = int((buf >= thr).sum().item())
            ts, _ = timed(lambda: ctx.score_range_compact(0, P, threshold=thr, capacity=kept))
            rec.update({"sparse_thr": thr, "sparse_kept": kept, "sparse_only_ms": ts, "sparse_over_dense": ts / t})
        out[f"override_long_tail_{frac}"] = rec
        print(json.dumps({f"override_long_tail_{frac}": rec}), flush=True)
        del buf
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/sparse_wide_bench.json").write_text(json.dumps(out, indent=1))
