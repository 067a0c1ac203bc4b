# ncu --set full of the C4 1x1 conv kernel (FP / dgrad launches) and the tiled max-pool backward
set -x
for k in "^k_conv_tc$:40:4" "k_pool_bwd_tile8:1:1"; do
  IFS=: read kre skip cnt <<< "$k"
  name=$(echo $kre | tr -dc 'a-z0-9_' | cut -c1-20)
  timeout 900 bash scripts/ncu_full.sh gpurun_out/c4ncu_$name "$kre" $skip $cnt --config c4 > gpurun_out/c4ncu_$name.txt 2>&1
  ncu -i gpurun_out/c4ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/c4ncu_$name.sass.csv 2>/dev/null
  ncu -i gpurun_out/c4ncu_$name.ncu-rep --page details --csv > gpurun_out/c4ncu_$name.details.csv 2>/dev/null
  rm -f gpurun_out/c4ncu_$name.ncu-rep
done
