#!/bin/bash
# A/B of the override kernels over every csrc/libnwap*.so (same box)
set -u
cd "$(dirname "$0")/.."
for lib in paper_2509_01654_b200/csrc/libnwap.so paper_2509_01654_b200/csrc/libnwap_*.so; do
  [ -f "$lib" ] || continue
  echo "== $(basename $lib .so)"
  NWAP_LIB=$lib timeout 300 python tools/ov_bench.py 100000 2>&1 | grep -v simple
done
