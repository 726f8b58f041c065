cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "matches_oracle" 2>&1 | tail -5
for v in 0 1; do
DPG_TG_RULE=$v timeout 300 python bench.py --steps 400 > gpurun_out/br_$v.json 2>gpurun_out/br_$v.err; echo "rc $?"; tail -2 gpurun_out/br_$v.err; python -c "
import json;d=json.load(open('gpurun_out/br_$v.json'));st=d['roofline']['stages_ms'];print('rule=$v',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if k.startswith('gs.')})"
done
timeout 300 python tools/graph_timeline.py 2>&1 | tail -26
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
