B=8 ncu --set full --clock-control none --import-source on -k "regex:k_conv_pair" -s 3 -c 1 -o gpurun_out/ncu_pair python scripts/microbench_layer.py 3,64,900,2400,7,2 2>&1 | tail -2
ncu -i gpurun_out/ncu_pair.ncu-rep --page raw --csv > gpurun_out/ncu_pair.raw.csv 2>&1
ncu -i gpurun_out/ncu_pair.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_pair.sass.csv 2>&1
ncu -i gpurun_out/ncu_pair.ncu-rep --page details --csv > gpurun_out/ncu_pair.details.csv 2>&1
