cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "matches_oracle" 2>&1 | tail -2
for v in 0 1; do
DPG_TG_RESB=$v timeout 300 python bench.py --steps 400 > gpurun_out/bres_$v.json 2>gpurun_out/bres_$v.err; tail -2 gpurun_out/bres_$v.err; python -c "
import json;d=json.load(open('gpurun_out/bres_$v.json'));st=d['roofline']['stages_ms'];print('resb=$v',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'dgrad' in k})"
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 --error-exitcode 99 python -m pytest -q -x -p no:cacheprovider "tests/test_gpu_step.py::test_step_matches_oracle" > gpurun_out/rc_resb.log 2>&1; echo "racecheck rc $?"; grep -E "SUMMARY|passed|failed" gpurun_out/rc_resb.log | tail -2
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 --error-exitcode 99 python -m pytest -q -x -p no:cacheprovider "tests/test_gpu_step.py::test_step_matches_oracle" > gpurun_out/sc_resb.log 2>&1; echo "synccheck rc $?"; grep -E "SUMMARY|passed|failed" gpurun_out/sc_resb.log | tail -2
