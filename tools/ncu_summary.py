#!/usr/bin/env python
"""Summarise an `ncu --set full --import-source on` capture of k_score_tiles into the text kept under
profiles/: the launch/pipe/stall metrics that matter for this kernel (raw page) and where the warp
time goes by code region (source page: DP matrix-row loops vs per-row / per-chunk code).

    python tools/ncu_summary.py gpurun_out/prof_tiles_c3.ncu-rep "header line" > profiles/rNN_ncu_....txt
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else ""
KEEP = re.compile(r"^(dram__bytes_(read|write)\.sum$|gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|gpu__time_duration.sum|"
                  r"launch__(block_size|grid_size|occupancy_limit_\w+|registers_per_thread)$|sm__cycles_elapsed.avg$|"
                  r"sm__inst_executed_pipe_(adu|alu|cbu|fma|lsu|uniform).avg.pct_of_peak_sustained_active|"
                  r"sm__warps_active.avg.pct_of_peak_sustained_active|smsp__average_warps_issue_stalled_\w+_per_issue_active.ratio|"
                  r"smsp__inst_executed.sum$|smsp__issue_active.avg.pct_of_peak_sustained_active|smsp__warps_eligible.avg.per_cycle_active)")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
print(f"# {title}")
print(f"# kernel: {vals[hdr.index('Kernel Name')]}")
for h, u, v in sorted(zip(hdr, units, vals)):
    if KEEP.match(h):
        print(f"{h:90s} {u:14s} {v}")

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
addr = [int(r[0], 16) for r in data]
text = [r[ix["Source"]].strip() for r in data]
samp = [float(r[ix["# Samples"]]) for r in data]
inst = [float(r[ix["Instructions Executed"]]) for r in data]
pos = {a: i for i, a in enumerate(addr)}
tot_s, tot_i = sum(samp), sum(inst)
inloop = [False] * len(data)
back = []
for i, t in enumerate(text):
    m = re.search(r"BRA\s+(?:P\d, )?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < addr[i] and tgt in pos:
            back.append((i - pos[tgt], pos[tgt], i))
for _, j, i in sorted(back):                       # innermost loops first: only they count as matrix-row loops
    if i - j < 200 and any("VIMNMX3" in text[k] for k in range(j, i + 1)) and not any(inloop[k] for k in range(j, i + 1)):
        for k in range(j, i + 1):
            inloop[k] = True
cell = re.compile(r"(VIMNMX3|VIADDMNMX|IMAD R\d+, R\d+, UR|VIADD R\d+, R\d+, UR|IADD3 R\d+, PT, PT, -R)")
first = min(k for k, f in enumerate(inloop) if f)
last = max(k for k, f in enumerate(inloop) if f)


def share(keys):
    return 100 * sum(samp[k] for k in keys) / tot_s, 100 * sum(inst[k] for k in keys) / tot_i


print("#")
print("# warp-time samples and executed instructions by code region (source page)")
regions = [
    ("DP matrix-row loops (all length bodies)", [k for k in range(len(data)) if inloop[k]]),
    ("  of which the four DP-cell instructions", [k for k in range(len(data)) if inloop[k] and cell.match(text[k])]),
    ("  of which loop control (LDS, pointer, test, move, branch)", [k for k in range(len(data)) if inloop[k] and not cell.match(text[k])]),
    ("before the bodies: unit/band/chunk set-up, column fetch, length dispatch", list(range(0, first))),
    ("inside the bodies, outside the matrix-row loops: row head, row init, select, emit", [k for k in range(first, last + 1) if not inloop[k]]),
    ("after the bodies: flush, end-of-band barrier, reductions", list(range(last + 1, len(data)))),
]
for name, keys in regions:
    s, i = share(keys)
    print(f"{name:85s} samples {s:5.1f} %   instructions {i:5.1f} %")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("# stall reasons, % of all samples: " + ", ".join(
    f"{h[6:]} {100 * sum(float(r[ix[h]] or 0) for r in data) / tot_s:.1f}" for h in stalls
    if sum(float(r[ix[h]] or 0) for r in data) / tot_s > 0.005))
by = {}
for k in range(len(data)):
    op = text[k].split()[1] if text[k].startswith("@") else text[k].split()[0]
    a = by.setdefault(op, [0.0, 0.0])
    a[0] += inst[k]
    a[1] += samp[k]
print("# executed instructions by opcode (>= 0.5 %): " + ", ".join(
    f"{op} {100 * v[0] / tot_i:.1f}" for op, v in sorted(by.items(), key=lambda x: -x[1][0]) if v[0] / tot_i >= 0.005))
