B=32 timeout -s KILL 120 python scripts/microbench_layer.py 256,256,56,56,3 128,128,112,112,3 512,512,28,28,3 2>&1 | tail -3
echo "rc=$?"
timeout -s KILL 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
