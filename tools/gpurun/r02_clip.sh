cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rules.py tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_norm.py -x -q 2>&1 | tail -3
for rep in 1 2; do
timeout 300 python bench.py --steps 400 > gpurun_out/bcl.json 2>gpurun_out/bcl.err; tail -2 gpurun_out/bcl.err; python -c "
import json;d=json.load(open('gpurun_out/bcl.json'));st=d['roofline']['stages_ms'];print(round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'clip' in k})"
done
