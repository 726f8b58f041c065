cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg_linear.py tests/test_gpu_rules.py -k "linear" > gpurun_out/lin_t.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/lin_t.log
for bn in 256 128; do DPG_TG_LIN_BN=$bn timeout 300 python bench.py --workload linear_t64 > gpurun_out/lin_bench_$bn.json 2> gpurun_out/lin_bench.err; echo "bench $bn rc $?"; python -c "
import json;d=json.load(open('gpurun_out/lin_bench_$bn.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('stages_ms'))"; done
DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=0 timeout 120 python tools/tg_trace_lin.py > gpurun_out/lintrace_0.txt 2>&1; grep tile gpurun_out/lintrace_0.txt | sed -n 2,4p
