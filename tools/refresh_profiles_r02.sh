#!/bin/bash
# Copy the artefacts of the last tools/gpu_r2c.sh session from gpurun_out/ (scratch) into profiles/ (tracked).
set -eu
cd "$(dirname "$0")/.."
R=${1:-r02}
cp gpurun_out/bench.json profiles/${R}_bench_c3.json
cp gpurun_out/bench_ref.json profiles/${R}_bench_reference_arm.json
cp gpurun_out/bench_torchrun1.json profiles/${R}_bench_torchrun_world1.json
cp gpurun_out/launches.csv profiles/${R}_launches_bench_default.csv
cp gpurun_out/pytest_gpu.log profiles/${R}_pytest_gpu.txt
grep -v "^{" gpurun_out/probes.log > profiles/${R}_probes.txt || true
python tools/ncu_summary.py gpurun_out/prof_tiles_c3.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:k_score_tiles -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-full-scale   (100,000 words, 4,999,950,000 pairs)" > profiles/${R}_ncu_k_score_tiles_c3.txt
python - "$R" <<'PY'
import json, re, sys
sys.path.insert(0, ".")
import bench
R = sys.argv[1]
f = f"profiles/{R}_ncu_k_score_tiles_c3.txt"
txt = open(f).read()
def val(name):
    m = re.search(rf"^{re.escape(name)}\s+(\S+)\s+(\S+)$", txt, re.M)
    unit, v = m.group(1), float(m.group(2))
    return int(v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[unit])
rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
out = json.load(open("profiles/traffic.json"))
out["100000"] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "algorithmic_bytes": 100000 * 99999 // 2,
                 "kernel": re.search(r"# kernel: (.*)", txt).group(1),
                 "kernel_source_digest": bench.kernel_source_digest(),
                 "source": f"{f} (ncu --set full --clock-control none)"}
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out["100000"], indent=1))
PY
