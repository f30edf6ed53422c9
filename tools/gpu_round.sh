#!/bin/bash
# One GPU-box session: tests, sanitizer, probes, bench, ncu.  Every step has its own timeout.
set -u
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/smoke.log
echo "== pytest gpu"; timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider --durations=6 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?"; tail -12 gpurun_out/pytest_gpu.log
echo "== probes"; timeout 120 python tools/probes.py > gpurun_out/probes.log 2>&1; tail -1 gpurun_out/probes.log | cut -c1-200
echo "== sanitizer"; timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_small.py 2300 > gpurun_out/memcheck.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/memcheck.log
echo "== racecheck"; timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_small.py 2100 > gpurun_out/racecheck.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/racecheck.log
echo "== bench C2-size"; timeout 300 python bench.py --words 20000 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "rc=$?"; tail -3 gpurun_out/bench_c2.err
echo "== bench default"; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
echo "== bench 600k words on one GPU (8 passes into one reused buffer)"; timeout 600 python bench.py --words 600000 --passes 8 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_600k.json 2> gpurun_out/bench_600k.err; echo "rc=$?"; cut -c1-260 gpurun_out/bench_600k.json; tail -3 gpurun_out/bench_600k.err
echo "== full-scale shards (C4, C5)"; timeout 600 python tools/fullscale_shards.py C4 > gpurun_out/fullscale_C4.log 2>&1; echo "rc=$?"; timeout 600 python tools/fullscale_shards.py C5 > gpurun_out/fullscale_C5.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/fullscale_C5.log | cut -c1-300
echo "== e2e breakdown"; timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; tail -8 gpurun_out/e2e_breakdown.txt
echo "== bench torchrun world=1"; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "rc=$?"; cut -c1-300 gpurun_out/bench_torchrun1.json; tail -3 gpurun_out/bench_torchrun1.err
echo "== bench reference"; timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?"; cut -c1-400 gpurun_out/bench_ref.json
echo "== ncu launches (default bench command)"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/launches.csv
echo "== ncu full C3"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_score_tiles -s 3 -c 1 -o gpurun_out/prof_tiles_c3 -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full_c3.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_full_c3.log | cut -c1-200
echo "== ncu full C2"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_tiles -s 3 -c 1 -o gpurun_out/prof_tiles -f python bench.py --words 20000 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "rc=$?"
ls -la gpurun_out
