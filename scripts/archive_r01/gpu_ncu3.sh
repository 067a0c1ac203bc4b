ncu --set full --clock-control none --import-source on -k "regex:k_conv_tc" -s 40 -c 4 -o gpurun_out/ncu_c2conv python bench.py --steps 1 --warmup 1 --no-baselines > /dev/null 2>&1
ncu -i gpurun_out/ncu_c2conv.ncu-rep --page raw --csv > gpurun_out/ncu_c2conv.raw.csv 2>&1
ncu -i gpurun_out/ncu_c2conv.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_c2conv.sass.csv 2>&1
ncu -i gpurun_out/ncu_c2conv.ncu-rep --page details --csv > gpurun_out/ncu_c2conv.details.csv 2>&1
python scripts/summarize_ncu.py gpurun_out/ncu_c2conv.raw.csv | grep -E "Name|duration|tensor_cycles_active.avg|lts__throughput|dram__bytes"
