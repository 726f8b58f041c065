cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/head_t.log 2>&1; echo "gpu suite rc $?"; tail -3 gpurun_out/head_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(round(d['value']),round(d['ms_per_step'],4),d['e2e']['value'],d['clocks'])"
