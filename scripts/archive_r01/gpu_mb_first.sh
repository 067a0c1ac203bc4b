B=32 timeout 300 python scripts/microbench_layer.py 3,64,56,224,3 3,64,224,224,3 2>&1 | tail -2
B=8 timeout 300 python scripts/microbench_layer.py 3,64,900,2400,7,2 2>&1 | tail -1
