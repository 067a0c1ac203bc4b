#!/bin/bash
# ncu evidence for the C4 bench step (1 GPU, under gpurun):
#   <tag>_launches.csv : every launch of one step (gpu__time_duration, --clock-control none)
#   <tag>_<name>.ncu-rep + .raw.csv + .txt : --set full of N launches of one kernel
# usage: bash scripts/ncu_c4.sh <tag> <kernel regex> <skip> <count> [one_step args]
TAG=$1; KRE=$2; SKIP=$3; CNT=$4; shift 4
mkdir -p gpurun_out
bash scripts/ncu_launches.sh gpurun_out/${TAG}_launches.csv "$@" > gpurun_out/${TAG}_launches.txt 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s "$SKIP" -c "$CNT" \
    -o gpurun_out/${TAG}_full python scripts/one_step.py "$@" > gpurun_out/${TAG}_full.log 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full.raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_full.sass.csv 2>/dev/null
python scripts/summarize_ncu.py gpurun_out/${TAG}_full.raw.csv > gpurun_out/${TAG}_full.txt
python scripts/sass_stalls.py gpurun_out/${TAG}_full.sass.csv > gpurun_out/${TAG}_full.stalls.txt 2>&1
