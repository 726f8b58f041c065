cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg_linear.py tests/test_gpu_rules.py -k "linear or clipped" > gpurun_out/ew_t.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/ew_t.log
for bn in 256 128 256 128; do
  DPG_TG_LIN_BN=$bn timeout 300 python bench.py --workload linear_t64 --steps 100 > gpurun_out/ew.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/ew.json'));r=d['roofline'];print('BN $bn lin',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"
done
