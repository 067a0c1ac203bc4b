#!/bin/bash
# One GPU session: pytest -m gpu, smoke, bench (default C4) -> gpurun_out/<tag>_*
# usage: bash scripts/gpu_run.sh <tag> [pytest -k expr or ""] [extra bench args...]
set -u
TAG=${1:-run}; K=${2:-}
EXTRA="${@:3}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -k "$K" > gpurun_out/${TAG}_pytest.txt 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.txt 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1200 python bench.py $EXTRA > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_pytest.txt
