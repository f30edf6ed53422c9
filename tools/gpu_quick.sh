#!/bin/bash
# Short GPU session: the new tests + a few bench lines.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
echo "== pytest new"; timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider --durations=8 -k "full_scale or c3_two" 2>&1 | tail -15
for v in simple packed3; do echo "== bench C2-size $v"; timeout 300 python bench.py --words 20000 --steps 3 --warmup 2 --no-cpu --no-e2e --variant $v 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), 'GCUPS', round(d['ms_per_step'],3),'ms')"; done
echo "== bench 600k single GPU is covered by the test timings above"
