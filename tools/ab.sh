#!/bin/bash
# A/B: benchmark every csrc/libnwap_*.so (and the default build) back to back on the same box.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for lib in paper_2509_01654_b200/csrc/libnwap.so paper_2509_01654_b200/csrc/libnwap_*.so; do
  [ -f "$lib" ] || continue
  tag=$(basename $lib .so)
  ok=$(NWAP_LIB=$lib timeout 200 python tools/sanitize_small.py 2300 2>&1 | grep -c " ok ")
  for variant in ${VARIANTS:-packed3}; do
    for words in 20000 100000; do
      steps=10; [ $words = 100000 ] && steps=3
      r=$(NWAP_LIB=$lib timeout 300 python bench.py --words $words --steps $steps --warmup 3 --no-cpu --no-e2e --variant $variant 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3))")
      echo "$tag parity_ok=$ok $variant words=$words GCUPS/ms: $r" | tee -a $out
    done
  done
done
