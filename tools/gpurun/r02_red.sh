cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py tests/test_gpu_step.py -k "clipped or oracle" > gpurun_out/red_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/red_t.log
for i in 1 2; do timeout 300 python bench.py --steps 400 > gpurun_out/red.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/red.json'));r=d['roofline'];print('cifar',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items() if k.startswith('csum')})"; done
