#!/bin/bash
# One ncu launch record per consumer kernel (time + DRAM bytes) while tools/consumers_bench.py runs.
# The threshold compaction launches come first (4 runs x 11 two-GiB slices), the normalised filter's after them.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/consumers_ncu_all.csv
for spec in "k_compact_count:1" "k_compact_scan:1" "k_compact_write:1" "k_payload_stats:1" "k_compact_count:45" "k_compact_write:45" "k_hist_normalized:1"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k "regex:^${k}" -s $s -c 1 --csv --log-file gpurun_out/_one.csv python tools/consumers_bench.py > /dev/null 2>&1
  grep -E '^"[0-9]' gpurun_out/_one.csv >> gpurun_out/consumers_ncu_all.csv
done
rm -f gpurun_out/_one.csv
wc -l gpurun_out/consumers_ncu_all.csv
