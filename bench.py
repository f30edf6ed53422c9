#!/usr/bin/env python
"""bench.py -- all-pairs Needleman-Wunsch scoring throughput on B200.

    python bench.py --gpus N --steps K --warmup W            (N>1: launched under torchrun)
    python bench.py --impl reference --gpus N --steps K --warmup W

A "step" is one complete all-pairs pass of the hot path over the synthetic
vocabulary: every rank scores its equal-work contiguous shard of the linear edge
range into a device-resident int8 buffer, with the summary statistics fused.

Workload (BASELINE.json): at N=1 this is configs[2], the 100,000-word
French-shaped vocabulary (4,999,950,000 pairs, scheme 1/-1/-2) -- the largest
configuration whose condensed output (5 GB) fits one GPU; configs[3] (600k words,
180 GB of output) does not.  Scaling is weak: N GPUs score round(100000*sqrt(N))
words so the pairs per GPU stay fixed.

Prints ONE JSON line (rank 0).  metric = DP cell updates per second (GCUPS);
pairs/s is reported beside it.  `e2e` is the same metric through the host-buffer
C-ABI call (word store H2D, scored payload D2H inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2509_01654_b200 import synth  # noqa: E402
from paper_2509_01654_b200.sharding import ShardStats, equal_work_bounds, reduce_stats, shard_of  # noqa: E402

METRIC = "all_pairs_nw_cell_updates_per_second"
UNIT = "GCUPS"
BASE_N = 100_000
SM_COUNT = 148


def workload(n_gpus: int, n_words: int | None, fixed_len: int = 0):
    n = n_words if n_words else int(round(BASE_N * math.sqrt(n_gpus)))
    ids, lens = synth.french_shaped(n)
    if fixed_len:      # diagnostic only: every word the same length (isolates length-mix effects)
        lens = np.full(n, fixed_len, dtype=np.uint8)
        ids = np.random.default_rng(1).integers(0, synth.ALPHABET, size=(n, fixed_len)).astype(np.uint8)
    scheme = synth.CONFIG_SCHEMES["C3"]
    name = (f"synthetic French-shaped vocabulary, n={n} words (configs[2] shape: length~clip(round(N(8.5,2.8)),1,24), "
            f"alphabet 40), scheme match/mismatch/gap={scheme}, all {n * (n - 1) // 2} pairs, int8 condensed output")
    return ids, lens, scheme, name


def range_cells(lens: np.ndarray, start: int, end: int) -> int:
    """Exact DP cells of linear range [start, end) from prefix sums (host ints)."""
    from paper_2509_01654_b200.triangle import col_of, row_of
    L = lens.astype(np.int64)
    n = L.size
    pre = np.concatenate([[0], np.cumsum(L)])
    roww = L * (pre[n] - pre[1:])
    rowpref = np.concatenate([[0], np.cumsum(roww)])
    P = n * (n - 1) // 2

    def before(idx):
        if idx <= 0:
            return 0
        if idx >= P:
            return int(rowpref[n - 1])
        r = row_of(idx, n)
        c = col_of(idx, n, r)
        return int(rowpref[r]) + int(L[r]) * int(pre[c] - pre[r + 1])

    return before(end) - before(start)


class ClockSampler:
    """nvidia-smi clock / throttle-reason sampler for the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "20", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for row in self.rows:
            f = [x.strip() for x in row.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2])); power.append(float(f[3]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


def cpu_reference_run(ids, lens, scheme, budget_s: float, threads: int):
    """Times the oracle port (oracle/nw_oracle.c: scalar DP per pair, pthread pool over contiguous
    chunks = the reference's fork pool) on evenly spaced 65,536-edge chunks of the workload."""
    from oracle import nw_oracle as orc
    n = len(lens)
    P = n * (n - 1) // 2
    ids32, len32 = ids.astype(np.int32), lens.astype(np.int32)
    sim = orc.similarity_matrix(scheme[0], scheme[1], int(ids.max()) + 1)
    chunk = 65536
    # calibrate on one chunk per thread, then size the sample for the budget
    t0 = time.perf_counter()
    orc.c_score_range(ids32, len32, sim, scheme[2], n, P // 2, min(P, P // 2 + chunk * threads), threads=threads)
    rate = chunk * threads / max(time.perf_counter() - t0, 1e-6)
    nchunks = int(max(threads, min((P + chunk - 1) // chunk, rate * budget_s / chunk)))
    nchunks = max(threads, (nchunks // threads) * threads)
    starts = [min(P - chunk, (P // nchunks) * k) for k in range(nchunks)] if P > chunk else [0]
    pairs = cells = 0
    import concurrent.futures as cf

    def one(s):
        e = min(P, s + chunk)
        orc.c_score_range(ids32, len32, sim, scheme[2], n, s, e, threads=1)
        return e - s, orc.cells_in_range(len32, n, s, e)

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:   # ctypes releases the GIL
        for p_, c_ in ex.map(one, starts):
            pairs += p_
            cells += c_
    dt = time.perf_counter() - t0
    return {"pairs": pairs, "cells": cells, "seconds": dt, "chunks": len(starts)}


def traffic_from_profile(n_words: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per k_score_tiles launch from the committed
    `ncu --set full` capture of this workload (profiles/traffic.json), or None."""
    f = ROOT / "profiles" / "traffic.json"
    if not f.exists():
        return None
    rec = json.loads(f.read_text()).get(str(n_words))
    return rec["dram_bytes_per_launch"] if rec else None


def numpy_port_rate(ids, lens, scheme, chunks: int = 2):
    """Single-process rate of the numpy restatement of the reference's batched engine."""
    from oracle import nw_oracle as orc
    n = len(lens)
    P = n * (n - 1) // 2
    ids32, len32 = ids.astype(np.int32), lens.astype(np.int32)
    sim = orc.similarity_matrix(scheme[0], scheme[1], int(ids.max()) + 1)
    t0 = time.perf_counter()
    pairs = 0
    for k in range(chunks):
        s = (P // (chunks + 1)) * (k + 1)
        e = min(P, s + 65536)
        orc.np_score_range(ids32, len32, sim, scheme[2], n, s, e)
        pairs += e - s
    return pairs / (time.perf_counter() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--words", type=int, default=0, help="override vocabulary size (default 100000*sqrt(gpus))")
    ap.add_argument("--variant", default="auto", choices=["auto", "packed", "packed3", "packed_sym", "simple"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the CPU baseline sample")
    ap.add_argument("--fixed-len", type=int, default=0, help="diagnostic: all words of this length")
    ap.add_argument("--passes", type=int, default=1,
                    help="score each rank's shard as this many equal-work sub-shards into one reused device buffer "
                         "(needed when the shard's int8 output exceeds HBM, e.g. --words 600000 --passes 8 on one GPU); "
                         "no e2e leg in this mode")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")

    ids, lens, scheme, wname = workload(args.gpus, args.words, args.fixed_len)
    n = len(lens)
    P = n * (n - 1) // 2
    cells_total = synth.total_cells(lens)
    host_threads = len(os.sched_getaffinity(0))

    # ------------------------------------------------------------------ reference arm (CPU)
    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        for it in range(args.warmup + args.steps):
            budget = max(1.0, args.cpu_seconds / max(1, args.steps)) if it >= args.warmup else 0.5
            r = cpu_reference_run(ids, lens, scheme, budget, host_threads)
            if it >= args.warmup:
                vals.append(r)
        cells = sum(v["cells"] for v in vals)
        pairs = sum(v["pairs"] for v in vals)
        secs = sum(v["seconds"] for v in vals)
        gcups = cells / secs / 1e9
        sample = (f"{vals[0]['chunks']} evenly spaced 65,536-edge chunks of the workload per step "
                  f"({pairs} pairs total), oracle port (scalar C DP per pair), extrapolated by cells")
        line = {
            "impl": "reference", "metric": METRIC, "value": gcups, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "pairs_per_s": pairs / secs,
            "config": {"workload": wname, "sampled": True},
            "cpu_baseline": {"value": gcups, "unit": UNIT, "cores": host_threads, "kind": "port", "sample": sample,
                             "pairs_per_s": pairs / secs,
                             "numpy_port_pairs_per_s_1proc": numpy_port_rate(ids, lens, scheme)},
            "e2e": {"value": gcups, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "projected_full_job_seconds": cells_total / (gcups * 1e9),
        }
        print(json.dumps(line))
        return

    # ------------------------------------------------------------------ our arm (GPU)
    import torch
    import torch.distributed as dist
    from paper_2509_01654_b200 import _native
    from paper_2509_01654_b200.engine import NwapContext, probe
    import paper_2509_01654_b200 as nw

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    L = _native.lib()
    sch = nw.ScoringScheme(*scheme)
    ctx = NwapContext(ids, lens, sch, device=local_rank)
    passes = max(1, args.passes)
    bounds = equal_work_bounds(lens, world * passes)
    s0, e0 = int(bounds[rank * passes]), int(bounds[(rank + 1) * passes])
    sub = [(int(bounds[rank * passes + k]), int(bounds[rank * passes + k + 1])) for k in range(passes)]
    shard_pairs = e0 - s0
    shard_cells = range_cells(lens, s0, e0)
    out = torch.empty(max(e - s for s, e in sub), dtype=torch.int8, device="cuda")
    if passes > 1:
        args.no_e2e = True

    def score_shard():
        """One step: this rank's whole shard (statistics accumulate over the sub-shards on the host side)."""
        if passes == 1:
            ctx.score_range(s0, e0, out, variant=args.variant, sync=False)
            return None
        acc = [0, 127, -128, 0]
        for s, e in sub:
            st = ctx.score_range(s, e, out, variant=args.variant)
            acc = [acc[0] + st[0], min(acc[1], st[1]), max(acc[2], st[2]), acc[3] + st[3]]
        return acc

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        score_shard()
    barrier()
    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()
    launches0 = L.nwap_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record()
    for k in range(args.steps):
        ev[k][0].record()
        acc = score_shard()
        ev[k][1].record()
    t_end.record()
    barrier()
    launches = L.nwap_launch_count() - launches0
    total_ms = t_start.elapsed_time(t_end)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    clocks = sampler.stop() if rank == 0 else None
    st = ctx.read_stats() if passes == 1 else (acc[0], acc[1], acc[2], acc[3])
    local = ShardStats(st[0], st[3], st[1], st[2])
    tmax = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    tot = reduce_stats(local)
    assert tot.count == P, f"scored {tot.count} of {P} pairs"
    ms_per_step = total_ms / args.steps
    gcups = cells_total / (ms_per_step * 1e-3) / 1e9
    pairs_per_s = P / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel (k_score_tiles): integer issue bound -------------
    roof = None
    if rank == 0:
        kern_ms = float(np.mean(step_ms))                 # `passes` k_score_tiles launches per step (+ tiny inits)
        # the packed cell's exact instruction mix (auto resolves to packed3 for a uniform scheme)
        mix_name, instr_per_cell, mix_desc = {
            "packed": ("mix_2alu_2imad", 4, "2 DPX + 2 IMAD"),
            "packed_sym": ("cell_2dpx_iadd3", 3, "2 DPX + IADD3"),
        }.get(args.variant, ("cell_2dpx_imad_iadd", 4, "2 DPX + IMAD + IADD"))
        ipc_mix, _ = probe(mix_name, 4000, local_rank)
        ipc_alu, _ = probe("vimnmx3_s16x2", 4000, local_rank)
        ipc_imad, _ = probe("imad", 4000, local_rank)
        sm_max = (clocks or {}).get("sm_max_mhz") or 1965.0
        sm_now = (clocks or {}).get("sm_mhz") or sm_max
        # instr_per_cell warp-instructions update one packed cell = 64 DP cells (32 lanes x s16x2)
        cells_per_instr = 64.0 / instr_per_cell
        peak_gcups = cells_per_instr * ipc_mix * SM_COUNT * sm_max * 1e6 / 1e9
        achieved = shard_cells / (kern_ms * 1e-3) / 1e9
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        roof = {
            "bound": "int-alu (DPX/IMAD issue; SURVEY 8(d): not hbm, not tensor)",
            "achieved": achieved, "peak": peak_gcups, "unit": "GCUPS", "frac": achieved / peak_gcups,
            "traffic": traffic_from_profile(n),
            "kernel": "k_score_tiles", "kernel_ms": kern_ms,
            "algorithmic_bytes": int(shard_pairs), "launches_per_step": passes,
            "peak_how": (f"live probe {mix_name}: {ipc_mix:.3f} warp-instr/clk/SM on the packed cell's own "
                         f"{instr_per_cell}-instruction mix ({mix_desc}) x {cells_per_instr:.2f} cells/instr x {SM_COUNT} SMs x "
                         f"{sm_max:.0f} MHz (clocks.max.sm); "
                         f"single-pipe probes: VIMNMX3.S16x2 {ipc_alu:.3f}, IMAD {ipc_imad:.3f} (both half-rate)"),
            "sm_mhz_under_load": sm_now,
            "frac_at_observed_clock": achieved / (cells_per_instr * ipc_mix * SM_COUNT * sm_now * 1e6 / 1e9),
            "hbm_write": {"achieved": shard_pairs / (kern_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                          "frac": shard_pairs / (kern_ms * 1e-3) / 1e9 / hbm_peak,
                          "peak_source": "measured" if peaks else "fallback"},
        }

    # ---- end to end through the host-buffer C-ABI call --------------------------------------
    e2e = None
    if not args.no_e2e:
        host = torch.empty(shard_pairs, dtype=torch.int8).pin_memory()
        ctx.close()
        del out
        torch.cuda.empty_cache()

        def e2e_step():
            with NwapContext(ids, lens, sch, device=local_rank) as c2:      # word store H2D
                return c2.score_range_host(s0, e0, host, variant=args.variant)   # payload D2H

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        assert r[3] == shard_pairs
        # plain pinned device->host copy on this box, for context: e2e is bounded by it (5 GB per step)
        probe_bytes = int(min(shard_pairs, 1 << 30))
        dsrc = torch.empty(probe_bytes, dtype=torch.int8, device="cuda")
        host[:probe_bytes].copy_(dsrc)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        host[:probe_bytes].copy_(dsrc)
        torch.cuda.synchronize()
        d2h_gbs = probe_bytes / (time.perf_counter() - t1) / 1e9
        del dsrc
        qpad = ((int(lens.max()) + 15) // 16) * 16
        e2e = {"value": cells_total / (dt / args.steps) / 1e9, "unit": UNIT,
               "pairs_per_s": P / (dt / args.steps), "ms_per_step": 1e3 * dt / args.steps,
               "h2d_bytes_per_step": int(n * qpad + n), "d2h_bytes_per_step": int(shard_pairs + 2080),
               "what": "NwapContext(host word store) + nwap_score_range_host into pinned host memory",
               "d2h_gbs_plain_copy": d2h_gbs,
               "d2h_bound_ms": 1e3 * shard_pairs / (d2h_gbs * 1e9)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu and world == 1:
        r = cpu_reference_run(ids, lens, scheme, args.cpu_seconds, host_threads)
        cpu = {"value": r["cells"] / r["seconds"] / 1e9, "unit": UNIT, "cores": host_threads, "kind": "port",
               "pairs_per_s": r["pairs"] / r["seconds"],
               "sample": (f"{r['chunks']} evenly spaced 65,536-edge chunks of the same workload ({r['pairs']} pairs, "
                          f"{r['seconds']:.1f} s), oracle/nw_oracle.c scalar DP on {host_threads} threads"),
               "numpy_port_pairs_per_s_1proc": numpy_port_rate(ids, lens, scheme)}

    line = {
        "metric": METRIC, "value": gcups, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "s16x2 (int16 cells, int8 output)", "data": "synthetic",
        "pairs_per_s": pairs_per_s,
        "config": {"workload": wname, "words": n, "pairs": P, "cells": cells_total, "variant": args.variant,
                   "l2": "output written per step (>= 5 GB per GPU) exceeds the 126 MB L2; the 3 MB word store is "
                         "L2/shared-memory resident by design",
                   "sharding": f"{world} equal-work contiguous shard(s)" + (f", each scored as {passes} sub-shards into one reused buffer" if passes > 1 else "")},
        "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu,
        "stats": {"sum": tot.sum, "min": tot.min, "max": tot.max, "count": tot.count},
        "step_ms": step_ms,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
