cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py tests/test_gpu_tg_linear.py tests/test_gpu_adapter.py tests/test_gpu_contexts.py > gpurun_out/side_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/side_t.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/side_f.log 2>&1; echo "full rc $?"; tail -1 gpurun_out/side_f.log
for i in 1 2; do timeout 300 python bench.py --workload linear_t64 > gpurun_out/side.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/side.json'));r=d['roofline'];print('lin',round(d['value']),round(d['ms_per_step'],4),round(d['e2e']['value']),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"; done
timeout 300 python bench.py --steps 300 > gpurun_out/side_c.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/side_c.json'));print('cifar',round(d['ms_per_step'],4))"
