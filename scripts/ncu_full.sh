#!/bin/bash
# One ncu --set full capture of the top kernels of a short bench run (1 GPU, under gpurun).
# usage: bash scripts/ncu_full.sh <out_basename> <kernel regex> <skip> <count> [bench args]
out=$1; kre=$2; skip=$3; cnt=$4; shift 4
ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c "$cnt" -o "$out" \
    python bench.py --steps 1 --warmup 1 --no-baselines "$@" > /dev/null 2>&1
ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>/dev/null
python scripts/summarize_ncu.py "$out.raw.csv"
