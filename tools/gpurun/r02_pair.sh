cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg.py tests/test_gpu_tg_linear.py tests/test_gpu_step.py > gpurun_out/pair_t.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/pair_t.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg3_cifar_b512 or cfg2 or cfg1" > gpurun_out/pair_f.log 2>&1; echo "full rc $?"; tail -2 gpurun_out/pair_f.log
for rep in 1 2; do
for lib in libdpg.so libdpg_p0.so; do
  DPG_LIB=$lib timeout 300 python bench.py --steps 400 > gpurun_out/pr.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/pr.json'));r=d['roofline'];print('$lib cifar',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items() if k.startswith(('fwd.conv','dgrad'))})"
done; done
for lib in libdpg.so libdpg_p0.so; do
  DPG_LIB=$lib timeout 300 python bench.py --workload linear_t64 --steps 100 > gpurun_out/pr.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/pr.json'));r=d['roofline'];print('$lib lin',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"
done
