cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py tests/test_gpu_tg_linear.py tests/test_gpu_step.py > gpurun_out/bias_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/bias_t.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2 or cfg4" > gpurun_out/bias_f.log 2>&1; echo "full rc $?"; tail -1 gpurun_out/bias_f.log
for i in 1 2; do timeout 300 python bench.py --workload linear_t64 > gpurun_out/bias.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bias.json'));r=d['roofline'];print('lin',round(d['value']),round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"; done
timeout 120 python tools/tg_trace_lin.py > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/tg_trace_lin.py 2>/dev/null | grep -E "gs_bias|narrow" | awk -F'","' '{print $5, $NF}' | cut -c1-120
