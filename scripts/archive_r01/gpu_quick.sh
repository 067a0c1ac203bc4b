# quick GPU check: parity tests, smoke, C2 + C4 bench lines (no baselines)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in "$@"; do
  timeout 600 python bench.py --config $cfg --no-baselines > gpurun_out/q_$cfg.log 2>&1
  tail -1 gpurun_out/q_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', round(d['value'],2), 'img/s ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'conv ms', round(r['ms_per_step'],3), 'wgrad', round(r['wgrad']['ms_per_step'],3), round(r['wgrad']['achieved'],1), 'other', round(r['other_ms_per_step'],3), d['clocks'])" || tail -5 gpurun_out/q_$cfg.log
done
