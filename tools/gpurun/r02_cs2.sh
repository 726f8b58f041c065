cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in 0 2; do
DPG_TG_CSUM=$v timeout 300 python bench.py --steps 400 > gpurun_out/bc.json 2>gpurun_out/bc.err; tail -2 gpurun_out/bc.err; python -c "
import json;d=json.load(open('gpurun_out/bc.json'));print('csum=$v',round(d['ms_per_step'],4))"
done
done
