#!/bin/bash
# Per-launch device times of one bench step (cold-cache, serialised: compare SHARES).
# usage (under gpurun): bash scripts/ncu_launches.sh <out.csv> [bench args]
out=${1:-gpurun_out/launches.csv}; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" \
    python bench.py --steps 1 --warmup 1 --no-baselines "$@" > /dev/null 2>&1
python scripts/summarize_launches.py "$out"
