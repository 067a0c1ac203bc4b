EPI=affine B=256 timeout 300 python scripts/microbench_layer.py 64,256,56,56,1 256,1024,14,14,1 2>&1 | tail -2
EPI=affine NBANDS=4 B=256 timeout 300 python scripts/microbench_layer.py 64,256,56,56,1 256,1024,14,14,1 2>&1 | tail -2
EPI=affine B=256 timeout 300 python scripts/microbench_layer.py 64,256,14,56,1 256,1024,4,14,1 2>&1 | tail -2
