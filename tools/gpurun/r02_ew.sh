cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg.py tests/test_gpu_tg_linear.py tests/test_gpu_step.py > gpurun_out/ew_t.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/ew_t.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/ew_f.log 2>&1; echo "full rc $?"; tail -2 gpurun_out/ew_f.log
for lib in libdpg.so libdpg_e4.so libdpg.so libdpg_e4.so; do
  DPG_LIB=$lib timeout 300 python bench.py --workload linear_t64 --steps 100 > gpurun_out/ew.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/ew.json'));r=d['roofline'];print('$lib lin',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"
done
DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=0 timeout 120 python tools/tg_trace_lin.py > gpurun_out/lintrace_0.txt 2>&1; grep tile gpurun_out/lintrace_0.txt | sed -n 2,3p
