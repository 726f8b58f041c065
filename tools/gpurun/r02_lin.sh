# T > 1 linear on the TMA core: parity tests, cfg2 bench, DPG_TG_LIN=0 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py -k "linear" > gpurun_out/lin_rules.log 2>&1; echo "rules rc $?"; tail -15 gpurun_out/lin_rules.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2" > gpurun_out/lin_cfg2.log 2>&1; echo "cfg2 rc $?"; tail -15 gpurun_out/lin_cfg2.log
timeout 300 python bench.py --workload linear_t64 > gpurun_out/lin_bench.json 2> gpurun_out/lin_bench.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/lin_bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('tensor'),r.get('stages_ms'))"
DPG_TG_LIN=0 timeout 300 python bench.py --workload linear_t64 > gpurun_out/lin_bench0.json 2> gpurun_out/lin_bench0.err; echo "bench0 rc $?"; python -c "
import json;d=json.load(open('gpurun_out/lin_bench0.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('stages_ms'))"
tail -5 gpurun_out/lin_bench.err
