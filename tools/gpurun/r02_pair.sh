cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 --error-exitcode 99 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg.py -k cluster > gpurun_out/rc_cluster.log 2>&1; echo "racecheck cluster rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/rc_cluster.log | tail -2
timeout 300 python -m pytest tests/test_gpu_tg.py -x -q 2>&1 | tail -2
timeout 300 python tools/tg_time.py 2>&1 | tail -9
for rep in 1 2; do
timeout 300 python bench.py --steps 400 > gpurun_out/bp.json 2>gpurun_out/bp.err; tail -2 gpurun_out/bp.err; python -c "
import json;d=json.load(open('gpurun_out/bp.json'));st=d['roofline']['stages_ms'];print(round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'fwd' in k or 'dgrad' in k})"
done
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
