cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tg.py -x -q 2>&1 | grep -E "^E |passed|failed|Error" | head -20
for v in 1 4; do
DPG_TG_CK=$v timeout 300 python bench.py --steps 300 > gpurun_out/bck_$v.json 2>gpurun_out/bck_$v.err; echo "rc $?"; tail -2 gpurun_out/bck_$v.err; python -c "
import json;d=json.load(open('gpurun_out/bck_$v.json'));st=d['roofline']['stages_ms'];print('ck=$v',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'dgrad' in k or 'fwd' in k})"
done
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -6
