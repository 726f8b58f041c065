cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_rules.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 400 > gpurun_out/bt.json 2>gpurun_out/bt.err; tail -2 gpurun_out/bt.err; python -c "
import json;d=json.load(open('gpurun_out/bt.json'));st=d['roofline']['stages_ms'];print(round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'fwd' in k})"
timeout 300 python bench.py --workload mnist_b64 --steps 400 > gpurun_out/btm.json 2>gpurun_out/btm.err; python -c "
import json;d=json.load(open('gpurun_out/btm.json'));print('mnist',round(d['ms_per_step'],4))"
