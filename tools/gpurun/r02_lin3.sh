cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py -k "linear or clipped" > gpurun_out/lin_rules.log 2>&1; echo "rules rc $?"; tail -2 gpurun_out/lin_rules.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/lin_cfg2.log 2>&1; echo "cfg2 rc $?"; tail -2 gpurun_out/lin_cfg2.log
timeout 300 python bench.py --workload linear_t64 > gpurun_out/lin_bench.json 2> gpurun_out/lin_bench.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/lin_bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('stages_ms'))"
DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=0 timeout 120 python tools/tg_trace_lin.py > gpurun_out/lintrace_0.txt 2>&1; grep tile gpurun_out/lintrace_0.txt | sed -n 2,5p
