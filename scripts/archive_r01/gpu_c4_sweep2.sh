for nb in 8 16 32; do
  timeout 900 python bench.py --config c4 --segments none --n-bands $nb > gpurun_out/bench_c4_none_nb$nb.log 2>&1; tail -1 gpurun_out/bench_c4_none_nb$nb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($nb, d['value'], d['memory'].get('reduction_x'), d['memory']['feature_map_bytes']/1e9, d['memory'].get('layerwise_feature_map_bytes',0)/1e9, d['config']['bands_per_segment'], d['memory']['plan'])"
done
