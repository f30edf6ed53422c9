#!/bin/bash
# Copy the artefacts of the last tools/gpu_round.sh session from gpurun_out/ (scratch) into profiles/ (tracked).
set -eu
cd "$(dirname "$0")/.."
R=${1:-r01}
cp gpurun_out/bench.json profiles/${R}_bench_c3.json
cp gpurun_out/bench_ref.json profiles/${R}_bench_reference_arm.json
cp gpurun_out/bench_torchrun1.json profiles/${R}_bench_torchrun_world1.json
cp gpurun_out/bench_600k.json profiles/${R}_bench_600k_one_gpu_8_passes.json
cp gpurun_out/launches.csv profiles/${R}_launches_bench_default.csv
cp gpurun_out/memcheck.log profiles/${R}_memcheck.txt
cp gpurun_out/racecheck.log profiles/${R}_racecheck.txt
cp gpurun_out/fullscale_C4.json profiles/${R}_fullscale_C4_one_gpu_8_shards.json
cp gpurun_out/fullscale_C5.json profiles/${R}_fullscale_C5_one_gpu_8_shards.json
cp gpurun_out/e2e_breakdown.txt profiles/${R}_e2e_breakdown.txt
grep -v "^{" gpurun_out/probes.log > profiles/${R}_probes.txt
python tools/ncu_summary.py gpurun_out/prof_tiles_c3.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:k_score_tiles -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e   (100,000 words, 4,999,950,000 pairs)" > profiles/${R}_ncu_k_score_tiles_c3.txt
python tools/ncu_summary.py gpurun_out/prof_tiles.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:k_score_tiles -s 3 -c 1 python bench.py --words 20000 --steps 1 --warmup 3 --no-cpu --no-e2e   (20,000 words, 199,990,000 pairs)" > profiles/${R}_ncu_k_score_tiles_c2.txt
python - "$R" <<'PY'
import json, re, sys
R = sys.argv[1]
out = {}
for n, f in (("100000", f"profiles/{R}_ncu_k_score_tiles_c3.txt"), ("20000", f"profiles/{R}_ncu_k_score_tiles_c2.txt")):
    txt = open(f).read()
    def val(name):
        m = re.search(rf"^{re.escape(name)}\s+(\S+)\s+(\S+)$", txt, re.M)
        unit, v = m.group(1), float(m.group(2))
        return int(v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[unit])
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    pairs = int(n) * (int(n) - 1) // 2
    kern = re.search(r"# kernel: (.*)", txt).group(1)
    out[n] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "algorithmic_bytes": pairs,
              "kernel": kern, "source": f"{f} (ncu --set full --clock-control none)"}
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
