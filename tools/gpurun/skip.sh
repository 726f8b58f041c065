cd $GRAFT_REPO_ROOT
for k in 0 1 2 4 8 3 5 6 7 9 10 12 14; do
  DPG_DBG_SKIP=$k python bench.py --no-cpu-baseline --steps 300 > gpurun_out/skip_$k.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/skip_$k.json')); print('skip $k', round(d['ms_per_step']*1000,1), 'us')"
done
