cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg.py tests/test_gpu_step.py tests/test_gpu_rules.py > gpurun_out/cew_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/cew_t.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg3_cifar_b512 or cfg1 or alternate" > gpurun_out/cew_f.log 2>&1; echo "full rc $?"; tail -1 gpurun_out/cew_f.log
for lib in libdpg.so libdpg_c4.so libdpg.so libdpg_c4.so; do
  DPG_LIB=$lib timeout 300 python bench.py --steps 400 > gpurun_out/cew.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/cew.json'));r=d['roofline'];print('$lib cifar',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items() if k.startswith(('fwd.conv','dgrad'))})"
done
for lib in libdpg.so libdpg_c4.so; do
  DPG_LIB=$lib timeout 300 python bench.py --workload mnist_b64 --steps 400 > gpurun_out/cew.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/cew.json'));print('$lib mnist',round(d['ms_per_step'],4))"
done
