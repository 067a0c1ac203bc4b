# launch lists (one step) + per-op CSVs for the given configs; tag = output prefix
tag=$1; shift
for cfg in "$@"; do
  bash scripts/ncu_launches.sh gpurun_out/${tag}_launches_$cfg.csv $cfg > gpurun_out/${tag}_launches_$cfg.txt 2>&1
  head -25 gpurun_out/${tag}_launches_$cfg.txt
  timeout 600 python bench.py --config $cfg --no-baselines --steps 3 --per-op-csv gpurun_out/${tag}_perop_$cfg.csv > /dev/null 2>&1
done
