timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp_merge" 2>&1 | tail -3
for cfg in c2 c4 c3; do
  for fl in 0 1; do
    LRCNN_BENCH_FP_MERGE=$fl timeout 600 python bench.py --config $cfg --no-baselines > gpurun_out/fm_${fl}_$cfg.json 2>gpurun_out/fm_${fl}_$cfg.err
    tail -1 gpurun_out/fm_${fl}_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg merge=$fl', round(d['value'],2), d['memory']['feature_map_bytes'])" || tail -3 gpurun_out/fm_${fl}_$cfg.err
  done
done
