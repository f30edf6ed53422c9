#!/bin/bash
# ncu --set full of the normalised consumers (one launch each) on a 2 GiB slice of a C5 shard
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_hist_norm_joint|k_compact_count|k_compact_write' -s 3 -c 3 -o gpurun_out/prof_consumers -f python tools/consumers_norm_only.py > gpurun_out/consumers_ncu_full.log 2>&1
echo rc=$?; tail -3 gpurun_out/consumers_ncu_full.log
