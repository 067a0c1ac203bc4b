for dbg in 0 1 2; do echo "DBG=$dbg"; LRCNN_TC_DBG=$dbg B=32 timeout -s KILL 120 python scripts/microbench_layer.py 256,256,56,56,3 512,512,28,28,3 2>&1 | tail -2; done
bash scripts/gpu_quick.sh c2 c3
