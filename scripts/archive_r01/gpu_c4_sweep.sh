# C4 memory/throughput sweep over the band count (per segment) + the layer-wise (COLUMN) peak
for nb in 4 8 16; do
  timeout 900 python bench.py --config c4 --n-bands $nb > gpurun_out/bench_c4_nb$nb.log 2>&1; tail -1 gpurun_out/bench_c4_nb$nb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($nb, d['value'], d['memory'].get('reduction_x'), d['memory']['feature_map_bytes']/1e9, d['memory'].get('layerwise_feature_map_bytes',0)/1e9, d['config']['bands_per_segment'])"
done
