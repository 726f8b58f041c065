cd $GRAFT_REPO_ROOT
DPG_TG_RULE=1 timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_step.py tests/test_gpu_tg.py > gpurun_out/r16_t.log 2>&1; echo "rule-on-core tests rc $?"; tail -1 gpurun_out/r16_t.log
DPG_TG_RULE=1 timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg3_cifar_b512" > gpurun_out/r16_f.log 2>&1; echo "rule-on-core fullsize rc $?"; tail -1 gpurun_out/r16_f.log
for v in 1 0 1 0; do DPG_TG_RULE=$v timeout 300 python bench.py --steps 400 > gpurun_out/r16.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r16.json'));r=d['roofline'];print('TG_RULE=$v',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items() if k.startswith(('gs.conv','csum.conv2d[2]'))})"; done
