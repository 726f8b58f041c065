cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tg.py -x -q 2>&1 | tail -2
timeout 300 python tools/tg_time.py 2>&1 | tail -9
timeout 300 python bench.py --steps 400 > gpurun_out/be.json 2>gpurun_out/be.err; tail -2 gpurun_out/be.err; python -c "
import json;d=json.load(open('gpurun_out/be.json'));st=d['roofline']['stages_ms'];print(round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'fwd' in k or 'dgrad' in k})"
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
