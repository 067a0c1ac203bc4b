# per-op CSV + bench lines (roofline with per-kernel bound) for the given configs
for cfg in "$@"; do
  timeout 600 python bench.py --config $cfg --no-baselines --per-op-csv gpurun_out/perop_$cfg.csv > gpurun_out/q_$cfg.json 2> gpurun_out/q_$cfg.err
  tail -1 gpurun_out/q_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', round(d['value'],2), 'img/s', {k: r[k] for k in ('bound','kernel','achieved','unit','frac','traffic')}); [print('   ', k['name'], round(k['ms_per_step'],3), k['bound'], round(k['achieved'],1), round(k['frac'],3)) for k in r['kernels']]" || tail -5 gpurun_out/q_$cfg.err
done
