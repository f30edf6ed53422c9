#!/bin/bash
# round 2 full GPU session: smoke, whole GPU suite, the driver's bench commands, launch list, ncu full capture
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/smoke.log
echo "== pytest gpu"; timeout 2400 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?"; tail -22 gpurun_out/pytest_gpu.log
echo "== bench default"; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
echo "== bench torchrun world=1"; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-full-scale > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "rc=$?"; cut -c1-300 gpurun_out/bench_torchrun1.json; tail -3 gpurun_out/bench_torchrun1.err
echo "== bench reference"; timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?"; cut -c1-600 gpurun_out/bench_ref.json
echo "== probes"; timeout 120 python tools/probes.py > gpurun_out/probes.log 2>&1; tail -1 gpurun_out/probes.log | cut -c1-200
echo "== ncu launches (default bench command)"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-full-scale > gpurun_out/ncu_launch.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/launches.csv
echo "== ncu full C3"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_score_tiles -s 3 -c 1 -o gpurun_out/prof_tiles_c3 -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-full-scale > gpurun_out/ncu_full_c3.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_full_c3.log | cut -c1-200
ls -la gpurun_out
