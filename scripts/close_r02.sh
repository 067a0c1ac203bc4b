#!/bin/bash
# Round-2 closing run on one GPU (under gpurun): full pytest -m gpu, smoke, bench lines (C4 default, C2,
# reference arm, training-mode BN C4 per block), then the profile bundle (scripts/profile_r02.sh).
tag=${1:-r02i}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 1200 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err
timeout 900 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
timeout 1500 python bench.py --config c4 --bn-train --segments block --steps 3 --warmup 3 > gpurun_out/${tag}_bench_c4_bn_block.json 2> gpurun_out/${tag}_bench_c4_bn_block.err
bash scripts/profile_r02.sh ${tag}
