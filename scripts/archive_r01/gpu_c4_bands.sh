# C4 band-count sweep: throughput and feature-map HBM (layer-wise reference: r01d_bench_c4.json)
for nb in 4 6 8 12 16; do
  timeout 600 python bench.py --config c4 --n-bands $nb --no-baselines > gpurun_out/c4b_$nb.json 2>gpurun_out/c4b_$nb.err
  tail -1 gpurun_out/c4b_$nb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['memory']; print('c4 bands $nb', round(d['value'],2), 'img/s fm GB', round(m['feature_map_bytes']/1e9,2), 'x', round(65174698592/m['feature_map_bytes'],2), d['config']['bands_per_segment'], d['config']['fp_bands_per_segment'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/c4b_$nb.err
done
