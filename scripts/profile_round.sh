#!/bin/bash
# Round profile bundle (1 GPU, under gpurun): launch lists of one C2 / C4 step, per-op CSVs,
# ncu --set full of the dominant conv and wgrad kernels of the C2 step, bench lines.
# usage: bash scripts/profile_round.sh <tag>
tag=${1:-rx}
for cfg in c2 c4; do
  bash scripts/ncu_launches.sh gpurun_out/${tag}_launches_$cfg.csv $cfg > gpurun_out/${tag}_launches_$cfg.txt 2>&1
  timeout 600 python bench.py --config $cfg --no-baselines --steps 3 --per-op-csv gpurun_out/${tag}_perop_$cfg.csv > /dev/null 2>&1
done
for k in "k_conv_tc2h:6:4" "k_wgrad_halo:6:3" "k_conv_tc2:40:2" "k_conv_halo_rb:6:2"; do
  IFS=: read kre skip cnt <<< "$k"
  name=$(echo $kre | tr -dc 'a-z0-9_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c $cnt \
      -o gpurun_out/${tag}_ncu_$name python bench.py --steps 1 --warmup 1 --no-baselines > /dev/null 2>&1
  ncu -i gpurun_out/${tag}_ncu_$name.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_ncu_$name.sass.csv 2>/dev/null
  python scripts/summarize_ncu.py gpurun_out/${tag}_ncu_$name.raw.csv > gpurun_out/${tag}_ncu_$name.txt
  rm -f gpurun_out/${tag}_ncu_$name.ncu-rep
done
timeout 900 python bench.py > gpurun_out/${tag}_bench_c2.json 2>gpurun_out/${tag}_bench_c2.err
timeout 900 python bench.py --config c4 --n-bands 16 > gpurun_out/${tag}_bench_c4.json 2>gpurun_out/${tag}_bench_c4.err
timeout 900 python bench.py --config c3 --no-baselines > gpurun_out/${tag}_bench_c3.json 2>gpurun_out/${tag}_bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>&1
tail -c 400 gpurun_out/${tag}_bench_c2.json; tail -c 300 gpurun_out/${tag}_bench_c4.json
