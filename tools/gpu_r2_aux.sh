#!/bin/bash
# round 2: consumers, override / table / wide / sparse-output benches (one GPU session)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
echo "== consumers"; timeout 600 python tools/consumers_bench.py > gpurun_out/consumers_bench.txt 2>&1; cat gpurun_out/consumers_bench.txt | tail -8
echo "== overrides"; timeout 300 python tools/ov_bench.py > gpurun_out/ov_bench.txt 2>&1; cat gpurun_out/ov_bench.txt
echo "== overrides 100k"; timeout 300 python tools/ov_bench.py 100000 > gpurun_out/ov_bench_100k.txt 2>&1; cat gpurun_out/ov_bench_100k.txt
echo "== tables"; timeout 300 python tools/tab_bench.py > gpurun_out/tab_bench.txt 2>&1; cat gpurun_out/tab_bench.txt
echo "== sparse / wide"; timeout 900 python tools/sparse_wide_bench.py > gpurun_out/sparse_wide_bench.txt 2>&1; cat gpurun_out/sparse_wide_bench.txt
