LRCNN_L2_CHUNK_MB=48 timeout 900 python -m pytest tests -m gpu -q -x -k "conditioned and (identity or bench_step or c4)" > gpurun_out/r02k_pytest_chunk.txt 2>&1; echo rc=$? >> gpurun_out/r02k_pytest_chunk.txt
for mb in 0 24 48 96; do
  LRCNN_L2_CHUNK_MB=$mb timeout 600 python bench.py --no-baselines --steps 8 > gpurun_out/r02k_bench_chunk$mb.json 2>&1
done
LRCNN_L2_CHUNK_MB=0 timeout 600 python bench.py --no-baselines --steps 8 > gpurun_out/r02k_bench_chunk0b.json 2>&1
