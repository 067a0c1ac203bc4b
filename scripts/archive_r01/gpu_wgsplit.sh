timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for m in 2 1; do
  for cfg in c3 c4; do
    LRCNN_WG_SPLIT_MUL=$m timeout 600 python bench.py --config $cfg --no-baselines > gpurun_out/wg_${m}_$cfg.json 2>/dev/null
    tail -1 gpurun_out/wg_${m}_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('mul $m $cfg', round(d['value'],2), [(k['name'], round(k['ms_per_step'],3)) for k in r['kernels'] if 'wgrad_tc' in k['name']])"
  done
done
