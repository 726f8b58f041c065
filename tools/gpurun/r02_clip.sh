cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py tests/test_gpu_tg_linear.py tests/test_gpu_adapter.py > gpurun_out/clip_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/clip_t.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/clip_f.log 2>&1; echo "full rc $?"; tail -1 gpurun_out/clip_f.log
for i in 1 2; do timeout 300 python bench.py --workload linear_t64 > gpurun_out/clip.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/clip.json'));r=d['roofline'];print('lin',round(d['value']),round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"; done
cp gpurun_out/clip.json gpurun_out/cfg_linear_t64.json
