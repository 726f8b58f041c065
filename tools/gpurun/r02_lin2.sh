cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py -k "linear" > gpurun_out/lin_rules.log 2>&1; echo "rules rc $?"; tail -3 gpurun_out/lin_rules.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/lin_cfg2.log 2>&1; echo "cfg2 rc $?"; tail -3 gpurun_out/lin_cfg2.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg.py tests/test_gpu_step.py > gpurun_out/lin_tgstep.log 2>&1; echo "tg+step rc $?"; tail -3 gpurun_out/lin_tgstep.log
timeout 300 python bench.py --workload linear_t64 > gpurun_out/lin_bench.json 2> gpurun_out/lin_bench.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/lin_bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('tensor'),r.get('stages_ms'))"
for k in 0 1; do DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=$k timeout 120 python tools/tg_trace_lin.py > gpurun_out/lintrace_$k.txt 2>&1; echo "trace $k rc $?"; head -30 gpurun_out/lintrace_$k.txt; tail -3 gpurun_out/lintrace_$k.txt; done
