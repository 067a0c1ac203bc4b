#!/bin/bash
# Closing verification on the final commit (1 GPU, under gpurun): pytest -m gpu, smoke, bench lines.
tag=${1:-r02k}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 1200 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err
timeout 900 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
