#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
echo "== pytest"; timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider --durations=5 ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -25
