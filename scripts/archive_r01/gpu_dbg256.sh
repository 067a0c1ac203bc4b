for dbg in 0 1 2 3; do
  echo "DBG=$dbg"; LRCNN_TC_DBG=$dbg B=32 timeout 300 python scripts/microbench_layer.py 256,256,56,56,3 128,128,112,112,3 2>&1 | tail -2
done
