cd $GRAFT_REPO_ROOT
for v in 1 0 1 0; do DPG_TG=$v timeout 300 python bench.py --workload mnist_b64 --steps 500 > gpurun_out/mn.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/mn.json'));r=d['roofline'];print('TG=$v',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items() if 'conv' in k})"; done
