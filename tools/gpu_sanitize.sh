#!/bin/bash
# compute-sanitizer memcheck + racecheck over every kernel family (tools/sanitize_small.py)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
echo "== plain"; timeout 300 python tools/sanitize_small.py 1500 > gpurun_out/sanitize_plain.log 2>&1; echo rc=$?; tail -4 gpurun_out/sanitize_plain.log
echo "== memcheck"; timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_small.py 1500 > gpurun_out/memcheck.log 2>&1; echo rc=$?; tail -3 gpurun_out/memcheck.log
echo "== racecheck"; timeout 2400 compute-sanitizer --tool racecheck python tools/sanitize_small.py 1100 > gpurun_out/racecheck.log 2>&1; echo rc=$?; tail -3 gpurun_out/racecheck.log
