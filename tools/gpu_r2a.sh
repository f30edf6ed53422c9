#!/bin/bash
# round 2, first GPU session: new kernels (sparse output, wide rows) + regression of the whole GPU suite + bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
echo "== new tests"; timeout 900 python -m pytest tests/test_gpu_sparse_wide.py -m gpu -q --tb=short -p no:cacheprovider -x 2>&1 | tail -30
echo "== full gpu suite"; timeout 1800 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/pytest_gpu.log
echo "== bench"; timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "rc=$?"; cut -c1-400 gpurun_out/bench_r2a.json; tail -3 gpurun_out/bench_r2a.err
