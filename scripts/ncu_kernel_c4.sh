#!/bin/bash
# ncu --set full of a few launches of one kernel inside one C4 training step (1 GPU, under gpurun).
# usage: bash scripts/ncu_kernel_c4.sh <out_basename> <kernel regex> [skip] [count] [config] [n_bands]
out=$1; kre=$2; skip=${3:-2}; cnt=${4:-1}; cfg=${5:-c4}; nb=${6:-8}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$kre" \
    -s "$skip" -c "$cnt" -o "$out" python scripts/one_step.py "$cfg" "$nb" > /dev/null 2>&1
ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>/dev/null
ncu -i "$out.ncu-rep" --page source --csv --print-source sass > "$out.sass.csv" 2>/dev/null
python scripts/summarize_ncu.py "$out.raw.csv" > "$out.txt"
python scripts/sass_stalls.py "$out.sass.csv" 25 > "$out.stalls.txt" 2>&1
rm -f "$out.ncu-rep"
