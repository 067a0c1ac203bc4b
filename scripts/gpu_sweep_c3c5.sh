#!/bin/bash
# BASELINE configs[2] (C3: ResNet-50 224^2 B=256, 2PS-H vs OverL-H at N in {2,4,7}) and configs[4]
# (C5: VGG-16 2048^2 B=16, band-height sweep for 2PS-H and OverL-H) -> gpurun_out/<tag>_<cfg>_*.json
TAG=${1:-sweep}
mkdir -p gpurun_out
for mode in 2ps overl; do
  for n in 2 4 7; do
    timeout 600 python bench.py --config c3 --mode $mode --n-bands $n --no-balanced --no-baselines --allow-overlap --steps 5 \
      > gpurun_out/${TAG}_c3_${mode}_${n}.json 2> gpurun_out/${TAG}_c3_${mode}_${n}.err
  done
done
for mode in 2ps overl; do
  for br in 8 16 32 64 128; do
    timeout 600 python bench.py --config c5 --mode $mode --band-rows $br --no-balanced --no-baselines --steps 3 \
      > gpurun_out/${TAG}_c5_${mode}_${br}.json 2> gpurun_out/${TAG}_c5_${mode}_${br}.err
  done
done
