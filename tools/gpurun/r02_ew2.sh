cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg.py tests/test_gpu_tg_linear.py tests/test_gpu_step.py > gpurun_out/ew_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/ew_t.log
DPG_LIB=libdpg_e16.so timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg_linear.py > gpurun_out/ew_t16.log 2>&1; echo "tests16 rc $?"; tail -1 gpurun_out/ew_t16.log
for lib in libdpg.so libdpg_e16.so libdpg.so libdpg_e16.so; do
  DPG_LIB=$lib timeout 300 python bench.py --workload linear_t64 --steps 100 > gpurun_out/ew.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/ew.json'));r=d['roofline'];print('$lib lin',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"
done
timeout 300 python bench.py --steps 300 > gpurun_out/ew.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/ew.json'));print('cifar',round(d['ms_per_step'],4))"
