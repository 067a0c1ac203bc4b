for db in 1 0; do
  echo "FUSE_DB=$db"
  EPI=affine LRCNN_FUSE_DB=$db B=256 timeout 300 python scripts/microbench_layer.py 64,256,14,56,1 256,64,14,56,1 256,1024,4,14,1 1024,256,4,14,1 2>&1 | tail -4
done
EPI=affine B=8 timeout 300 python scripts/microbench_layer.py 64,256,225,600,1 256,64,225,600,1 2>&1 | tail -2
