# ncu --set full of the C3 1x1 wgrad (k_wgrad_tc) and the C4 stem kernels
set -x
timeout 900 bash scripts/ncu_full.sh gpurun_out/c3ncu_wgrad "^k_wgrad_tc$" 40 3 --config c3 > gpurun_out/c3ncu_wgrad.txt 2>&1
ncu -i gpurun_out/c3ncu_wgrad.ncu-rep --page source --csv --print-source sass > gpurun_out/c3ncu_wgrad.sass.csv 2>/dev/null
ncu -i gpurun_out/c3ncu_wgrad.ncu-rep --page details --csv > gpurun_out/c3ncu_wgrad.details.csv 2>/dev/null
rm -f gpurun_out/c3ncu_wgrad.ncu-rep
timeout 900 bash scripts/ncu_full.sh gpurun_out/c4ncu_stem "k_conv_pair|k_wgrad_im2col|k_pool3s2_bwd" 0 3 --config c4 > gpurun_out/c4ncu_stem.txt 2>&1
ncu -i gpurun_out/c4ncu_stem.ncu-rep --page source --csv --print-source sass > gpurun_out/c4ncu_stem.sass.csv 2>/dev/null
ncu -i gpurun_out/c4ncu_stem.ncu-rep --page details --csv > gpurun_out/c4ncu_stem.details.csv 2>/dev/null
rm -f gpurun_out/c4ncu_stem.ncu-rep
