for db in 1 0; do
  echo "FUSE_DB=$db"
  EPI=affine LRCNN_FUSE_DB=$db B=8 timeout 300 python scripts/microbench_layer.py 128,128,35,300,3 128,128,112,300,3 64,64,56,600,3 64,64,225,600,3 2>&1 | tail -4
done
