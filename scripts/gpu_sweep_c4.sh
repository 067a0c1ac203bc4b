#!/bin/bash
# C4 segment / band sweep (no baselines) -> gpurun_out/<tag>_sweep_<segs>_<n>.json
TAG=${1:-sweep}
mkdir -p gpurun_out
for cfg in "pool 8" "pool 4" "3 16" "3 32" "none 16" "none 32" "34 16"; do
  set -- $cfg
  timeout 600 python bench.py --no-baselines --segments $1 --n-bands $2 --steps 8 > gpurun_out/${TAG}_sweep_$1_$2.json 2> gpurun_out/${TAG}_sweep_$1_$2.err
done
