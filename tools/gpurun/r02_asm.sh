cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg_linear.py tests/test_gpu_rules.py -k "linear or clipped" > gpurun_out/asm_t.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/asm_t.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/asm_f.log 2>&1; echo "full rc $?"; tail -1 gpurun_out/asm_f.log
for lib in libdpg.so libdpg_a0.so libdpg.so libdpg_a0.so; do
  DPG_LIB=$lib timeout 300 python bench.py --workload linear_t64 --steps 100 > gpurun_out/asm.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/asm.json'));r=d['roofline'];print('$lib lin',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"
done
