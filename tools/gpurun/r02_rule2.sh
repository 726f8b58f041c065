cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tg.py tests/test_gpu_step.py -x -q -k "matches_oracle or tg_gemm" 2>&1 | tail -2
DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=5 timeout 120 python tools/tg_trace_step.py 2>&1 | tail -8
for v in 0 1; do
DPG_TG_RULE=$v timeout 300 python bench.py --steps 400 > gpurun_out/br_$v.json 2>gpurun_out/br_$v.err; echo "rc $?"; tail -2 gpurun_out/br_$v.err; python -c "
import json;d=json.load(open('gpurun_out/br_$v.json'));st=d['roofline']['stages_ms'];print('rule=$v',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if k.startswith('gs.') or 'fwd' in k or 'dgrad' in k})"
done
