B=8 ncu --set full --clock-control none --import-source on -k "regex:k_conv_tc" -s 6 -c 1 -o gpurun_out/ncu_1x1_fp python scripts/microbench_layer.py 64,256,225,600,1 2>&1 | tail -5
ncu -i gpurun_out/ncu_1x1_fp.ncu-rep --page raw --csv > gpurun_out/ncu_1x1_fp.raw.csv 2>&1
ncu -i gpurun_out/ncu_1x1_fp.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_1x1_fp.sass.csv 2>&1
ncu -i gpurun_out/ncu_1x1_fp.ncu-rep --page details --csv > gpurun_out/ncu_1x1_fp.details.csv 2>&1
ls -la gpurun_out
