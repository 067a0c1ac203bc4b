for ew in 0 1; do for dbg in 0 1 2 3; do
  echo "EPI_W=$ew DBG=$dbg"
  LRCNN_EPI_W=$ew LRCNN_TC_DBG=$dbg B=8 timeout 300 python scripts/microbench_layer.py 64,256,225,600,1 256,1024,57,150,1 2>&1 | tail -2
done; done
