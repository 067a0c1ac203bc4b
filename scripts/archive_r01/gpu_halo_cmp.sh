for h in 0 1; do
echo "LRCNN_HALO=$h"
LRCNN_HALO=$h B=32 timeout 300 python scripts/microbench_layer.py 64,128,112,112,3 128,128,112,112,3 128,256,56,56,3 256,256,56,56,3 512,512,28,28,3 512,512,14,14,3 2>&1 | tail -6
done
