#!/bin/bash
# Round profile bundle (1 GPU, under gpurun): launch lists of one C2 / C4 step, per-op CSVs,
# ncu --set full of the dominant kernels (C2: CTA-pair halo conv, 3x3 wgrad; C4: 1x1 conv, 1x1
# wgrad, stem, max-pool backward), profiles/traffic.json, bench lines, the GPU tests.
# usage: bash scripts/profile_round.sh <tag>
tag=${1:-rx}
for cfg in c2 c4; do
  bash scripts/ncu_launches.sh gpurun_out/${tag}_launches_$cfg.csv $cfg > gpurun_out/${tag}_launches_$cfg.txt 2>&1
done
for cfg in c2 c3 c4; do
  timeout 600 python bench.py --config $cfg --no-baselines --steps 3 --per-op-csv gpurun_out/${tag}_perop_$cfg.csv > /dev/null 2>&1
done
caps=""
for k in "c2:k_conv_tc2h:6:4" "c2:k_wgrad_halo:6:3" "c4:^k_conv_tc$:40:4" "c4:^k_wgrad_tc$:30:3" "c4:k_conv_pair:1:1" "c4:k_pool3s2_bwd:0:1"; do
  IFS=: read cfg kre skip cnt <<< "$k"
  name=${cfg}_$(echo $kre | tr -dc 'a-z0-9_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c $cnt \
      -o gpurun_out/${tag}_ncu_$name python bench.py --config $cfg --steps 1 --warmup 1 --no-baselines > /dev/null 2>&1
  ncu -i gpurun_out/${tag}_ncu_$name.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_ncu_$name.sass.csv 2>/dev/null
  python scripts/summarize_ncu.py gpurun_out/${tag}_ncu_$name.raw.csv > gpurun_out/${tag}_ncu_$name.txt
  python scripts/sass_stalls.py gpurun_out/${tag}_ncu_$name.sass.csv 20 > gpurun_out/${tag}_ncu_$name.stalls.txt 2>&1
  rm -f gpurun_out/${tag}_ncu_$name.ncu-rep gpurun_out/${tag}_ncu_$name.sass.csv
  caps="$caps gpurun_out/${tag}_ncu_$name.raw.csv"
done
python scripts/make_traffic.py gpurun_out/${tag}_traffic.json $caps > /dev/null
cp gpurun_out/${tag}_traffic.json profiles/traffic.json
timeout 900 python bench.py > gpurun_out/${tag}_bench_c2.json 2>gpurun_out/${tag}_bench_c2.err
timeout 900 python bench.py --config c4 > gpurun_out/${tag}_bench_c4.json 2>gpurun_out/${tag}_bench_c4.err
timeout 900 python bench.py --config c4 --n-bands 4 --no-baselines > gpurun_out/${tag}_bench_c4_4.json 2>gpurun_out/${tag}_bench_c4_4.err
timeout 900 python bench.py --config c3 --no-baselines > gpurun_out/${tag}_bench_c3.json 2>gpurun_out/${tag}_bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>&1
tail -c 300 gpurun_out/${tag}_bench_c2.json; tail -c 300 gpurun_out/${tag}_bench_c4.json
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/${tag}_pytest_gpu.txt
cat gpurun_out/${tag}_pytest_gpu.txt
