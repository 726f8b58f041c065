cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tg.py -q -rf -x 2>&1 | grep -E "^E " | head
timeout 600 python bench.py --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -3 gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['stages_ms'])"
