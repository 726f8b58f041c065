cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do
DPG_TG_CSUM=$v timeout 300 python bench.py --steps 300 > gpurun_out/bcs_$v.json 2>gpurun_out/bcs_$v.err; echo "rc $?"; tail -2 gpurun_out/bcs_$v.err; python -c "
import json;d=json.load(open('gpurun_out/bcs_$v.json'));st=d['roofline']['stages_ms'];print('csum=$v',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'csum' in k})"
done
for s in 2 3 4 8; do
DPG_TG_CSUM_SPL=$s timeout 300 python bench.py --steps 300 > gpurun_out/bcs_s$s.json 2>gpurun_out/bcs_s$s.err; python -c "
import json;d=json.load(open('gpurun_out/bcs_s$s.json'));st=d['roofline']['stages_ms'];print('spl=$s',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'csum' in k})"
done
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -6
