cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -rf -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_full.log | head -20
timeout 600 python bench.py --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['stages_ms'])"
