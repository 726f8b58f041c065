cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/diag_parity.py cifar_b512 64 1.48 2>&1 | tail -11 | head -3
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_rules.py tests/test_golden.py tests/test_gpu_norm.py -q 2>&1 | tail -4
timeout 600 python bench.py --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -3 gpurun_out/bench.err; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step']);st=d['roofline']['stages_ms'];print({k:round(v*1e3,1) for k,v in st.items()})"
