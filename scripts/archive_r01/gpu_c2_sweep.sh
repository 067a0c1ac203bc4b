# C2 band-count sweep: throughput vs feature-map memory (2PS-H per pool, balanced bands), plus whole-net 2PS and OverL
for nb in 1 2 4 8 16; do
  timeout 300 python bench.py --n-bands $nb > gpurun_out/c2_nb$nb.json 2>/dev/null
  tail -1 gpurun_out/c2_nb$nb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['memory']; print('2ps-h nb=$nb', round(d['value'],1), d['config']['bands_per_segment'], round(m['feature_map_bytes']/1e9,3), round(m.get('reduction_x',0),2))"
done
for nb in 4 8; do
  timeout 300 python bench.py --segments none --n-bands $nb > gpurun_out/c2_none_nb$nb.json 2>/dev/null
  tail -1 gpurun_out/c2_none_nb$nb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['memory']; print('2ps whole nb=$nb', round(d['value'],1), d['config']['bands_per_segment'], round(m['feature_map_bytes']/1e9,3), round(m.get('reduction_x',0),2))"
  timeout 300 python bench.py --mode overl --n-bands $nb > gpurun_out/c2_overl_nb$nb.json 2>/dev/null
  tail -1 gpurun_out/c2_overl_nb$nb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['memory']; print('overl-h nb=$nb', round(d['value'],1), d['config']['bands_per_segment'], round(m['feature_map_bytes']/1e9,3), round(m.get('reduction_x',0),2))"
done
timeout 300 python bench.py --mode column > gpurun_out/c2_column.json 2>/dev/null
tail -1 gpurun_out/c2_column.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['memory']; print('column', round(d['value'],1), round(m['feature_map_bytes']/1e9,3))"
