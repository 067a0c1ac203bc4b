#!/bin/bash
# Round-2 evidence bundle (1 GPU, under gpurun) -> gpurun_out/<tag>_*:
#   launch lists of one C4 / C2 step (ncu gpu__time_duration, serialised, cold: compare shares),
#   per-op CSVs, DRAM bytes of EVERY launch of the dominant kernels in one C4 step (traffic.json),
#   ncu --set full of a few launches of the top kernels (+ stall summaries), bench lines.
# usage: bash scripts/profile_r02.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
bash scripts/ncu_launches.sh gpurun_out/${tag}_launches_c4.csv c4 8 > gpurun_out/${tag}_launches_c4.txt 2>&1
bash scripts/ncu_launches.sh gpurun_out/${tag}_launches_c2.csv c2 4 > gpurun_out/${tag}_launches_c2.txt 2>&1
for cfg in c2 c4; do
  timeout 600 python bench.py --config $cfg --no-baselines --steps 3 --per-op-csv gpurun_out/${tag}_perop_$cfg.csv \
    > gpurun_out/${tag}_perop_$cfg.json 2>&1
done
# DRAM traffic of every launch of the top kernels in one C4 step
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --profile-from-start off --kernel-name-base demangled \
    -k "regex:k_conv_tc|k_wgrad_tc|k_dwgrad_pw|k_conv_halo_rb|k_conv_pair|k_bneck_fwd|k_wgrad_im2col|k_wgrad_halo|k_pool3s2_bwd" -o gpurun_out/${tag}_traffic_c4 \
    python scripts/one_step.py c4 8 > gpurun_out/${tag}_traffic_c4.log 2>&1
ncu -i gpurun_out/${tag}_traffic_c4.ncu-rep --page raw --csv > gpurun_out/${tag}_traffic_c4.raw.csv 2>/dev/null
rm -f gpurun_out/${tag}_traffic_c4.ncu-rep
python scripts/make_traffic.py gpurun_out/${tag}_traffic.json gpurun_out/${tag}_traffic_c4.raw.csv > /dev/null
# --set full of a few launches of the top kernels
for k in "k_conv_tc<.int.256, .int.64, .int.8>:20:3" "k_conv_tc2<.int.256>:20:3" "k_wgrad_tc<.int.256>:20:3" "k_bneck_fwd:2:2" \
         "k_dwgrad_pw<.int.256, .int.64>:4:2" "k_dwgrad_pw<.int.64, .int.256>:4:2" "k_conv_pair:1:1"; do
  IFS=: read kre skip cnt <<< "$k"
  name=$(echo "$kre" | tr -dc 'a-z0-9_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$kre" \
      -s $skip -c $cnt -o gpurun_out/${tag}_ncu_$name python scripts/one_step.py c4 8 > /dev/null 2>&1
  ncu -i gpurun_out/${tag}_ncu_$name.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_ncu_$name.sass.csv 2>/dev/null
  python scripts/summarize_ncu.py gpurun_out/${tag}_ncu_$name.raw.csv > gpurun_out/${tag}_ncu_$name.txt
  python scripts/sass_stalls.py gpurun_out/${tag}_ncu_$name.sass.csv 20 > gpurun_out/${tag}_ncu_$name.stalls.txt 2>&1
  rm -f gpurun_out/${tag}_ncu_$name.ncu-rep gpurun_out/${tag}_ncu_$name.sass.csv
done
