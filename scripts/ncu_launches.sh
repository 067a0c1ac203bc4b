#!/bin/bash
# Per-launch device times of ONE training step (the step replayed from its CUDA graph;
# ncu serialises launches and runs them cold: compare SHARES, not the absolute sum).
# usage (under gpurun): bash scripts/ncu_launches.sh <out.csv> [config] [n_bands]
out=${1:-gpurun_out/launches.csv}; shift
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file "$out" \
    python scripts/one_step.py "$@" > /dev/null 2>&1
python scripts/summarize_launches.py "$out"
