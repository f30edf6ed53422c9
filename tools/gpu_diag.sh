#!/bin/bash
set -u
cd "$(dirname "$0")/.."
for lib in paper_2509_01654_b200/csrc/libnwap.so paper_2509_01654_b200/csrc/libnwap_*.so; do
  [ -f "$lib" ] || continue
  echo "== $(basename $lib)  parity: $(NWAP_LIB=$lib timeout 200 python tools/sanitize_small.py 2300 2>&1 | grep -c ' ok ')"
  for L in 4 8 12 16; do
    r=$(NWAP_LIB=$lib timeout 300 python bench.py --words 30000 --fixed-len $L --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), 'GCUPS', round(d['ms_per_step'],3),'ms')")
    echo "fixed_len=$L: $r"
  done
  for W in 20000 100000; do
    r=$(NWAP_LIB=$lib timeout 300 python bench.py --words $W --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), 'GCUPS', round(d['ms_per_step'],3),'ms')")
    echo "french $W: $r"
  done
done
