# ncu --set full of the C4 (ResNet-50 3600x2400) HBM-bound kernels: 1x1 wgrad, 1x1 conv, pool backward, stem
set -x
for k in "k_wgrad_tc:30:2" "k_conv_tc<:60:2" "k_pool3s2_bwd|pool.*bwd:1:1" "k_conv_pair:1:1" "k_acc_gate:10:1"; do
  IFS=: read kre skip cnt <<< "$k"
  name=$(echo $kre | tr -dc 'a-z0-9_' | cut -c1-20)
  timeout 900 bash scripts/ncu_full.sh gpurun_out/c4ncu_$name "$kre" $skip $cnt --config c4 > gpurun_out/c4ncu_$name.txt 2>&1
  ncu -i gpurun_out/c4ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/c4ncu_$name.sass.csv 2>/dev/null
  rm -f gpurun_out/c4ncu_$name.ncu-rep
done
