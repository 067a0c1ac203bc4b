#!/bin/bash
# ncu --set full of one kernel launched by scripts/microbench_layer.py (1 GPU, under gpurun).
# usage: bash scripts/ncu_layer.sh <out_basename> <kernel regex> <shape> [skip]
out=$1; kre=$2; shape=$3; skip=${4:-3}
B=${B:-32} ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 1 -o "$out" \
    python scripts/microbench_layer.py "$shape" > /dev/null 2>&1
ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>/dev/null
ncu -i "$out.ncu-rep" --page source --csv --print-source sass > "$out.sass.csv" 2>/dev/null
python scripts/summarize_ncu.py "$out.raw.csv"
