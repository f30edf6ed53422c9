#!/bin/bash
# ncu --set full records of the override-scheme kernels at 20,000 words (tools/ov_bench.py): launch 5 = sparse-correction
# cell on the frequent set... the bench launches, in order: uniform x2, rare packed3 x2, rare tab x2, frequent packed3 x2,
# frequent tab x2, generic x2
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "ov:k_score_tiles:7" "tab:k_score_tiles:9" "simple:k_score_simple:1"; do
  name=${spec%%:*}; rest=${spec#*:}; k=${rest%%:*}; s=${rest##*:}
  timeout 600 ncu --set full --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/prof_$name -f python tools/ov_bench.py 20000 > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
ls -la gpurun_out
