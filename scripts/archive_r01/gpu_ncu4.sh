B=32 ncu --set full --clock-control none --import-source on -k "regex:k_conv_pair" -s 3 -c 1 -o gpurun_out/ncu_pair1 python scripts/microbench_layer.py 3,64,56,224,3 > /dev/null 2>&1
ncu -i gpurun_out/ncu_pair1.ncu-rep --page raw --csv > gpurun_out/ncu_pair1.raw.csv 2>&1
ncu -i gpurun_out/ncu_pair1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_pair1.sass.csv 2>&1
