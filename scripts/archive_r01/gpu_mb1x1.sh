# 1x1 memory-bound conv microbenchmarks + one ncu capture of the FP kernel
B=8 timeout 300 python scripts/microbench_layer.py 64,256,225,600,1 256,64,225,600,1 64,64,225,600,3 256,1024,57,150,1 1024,256,57,150,1 2>&1 | tail -6
B=8 bash scripts/ncu_layer.sh gpurun_out/ncu_1x1_fp 'k_conv_tc<256' 64,256,225,600,1 3 2>&1 | tail -25
