set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
timeout 600 python bench.py --config c4 --no-baselines > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log
timeout 600 python bench.py --config c3 --no-baselines > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log
