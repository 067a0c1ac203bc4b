for dbg in 0 1 2 3; do echo "DBG=$dbg"; LRCNN_TC_DBG=$dbg B=8 timeout -s KILL 120 python scripts/microbench_layer.py 64,256,225,600,1 256,64,225,600,1 128,512,113,300,1 2>&1 | tail -3; done
