#!/bin/bash
# Fixed-length diagnostics (every word of length L) and the default bench, one line each.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/fixedlen.txt; : > $out
for L in ${LENS:-4 8 12 16 21 28 32}; do
  python bench.py --words 40000 --fixed-len $L --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('fixed-len $L GCUPS/ms:', round(d['value']), round(d['ms_per_step'],3))" | tee -a $out
done
python bench.py --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('default bench GCUPS', round(d['value']), 'step_ms', [round(x,2) for x in d['step_ms']], 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3))" | tee -a $out
