set -x
timeout 900 python bench.py --config c3 --bn-train --steps 5 --warmup 3 --no-baselines > gpurun_out/bnb_c3.json 2> gpurun_out/bnb_c3.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-baselines > gpurun_out/bnb_c3_frozen.json 2> gpurun_out/bnb_c3_frozen.err
timeout 1200 python bench.py --config c4 --bn-train --segments block --steps 3 --warmup 3 --no-baselines > gpurun_out/bnb_c4_block.json 2> gpurun_out/bnb_c4_block.err
timeout 1200 python bench.py --config c4 --bn-train --steps 3 --warmup 3 > gpurun_out/bnb_c4_stage.json 2> gpurun_out/bnb_c4_stage.err
