cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -x -q 2>&1 | tail -2
timeout 300 python tools/graph_timeline.py 2>&1 | tail -24
for rep in 1 2; do
timeout 300 python bench.py --steps 400 > gpurun_out/bs.json 2>gpurun_out/bs.err; tail -2 gpurun_out/bs.err; python -c "
import json;d=json.load(open('gpurun_out/bs.json'));print('bench',round(d['ms_per_step'],4), d['value'])"
done
