cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DPG_TG_RULE1=1 timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "matches_oracle" 2>&1 | tail -3
for v in 0 1; do
DPG_TG_RULE1=$v timeout 300 python bench.py --steps 400 > gpurun_out/br1.json 2>gpurun_out/br1.err; tail -2 gpurun_out/br1.err; python -c "
import json;d=json.load(open('gpurun_out/br1.json'));st=d['roofline']['stages_ms'];print('rule1=$v',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if k.startswith('gs.')})"
done
