cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck; do
  echo "=== $tool: tests/test_gpu_tg.py + step/rules subset"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest -q -x -p no:cacheprovider \
    tests/test_gpu_tg.py "tests/test_gpu_step.py::test_step_matches_oracle" tests/test_gpu_rules.py -k "not embedding_large" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc $?"; grep -E "ERROR SUMMARY|passed|failed|error" gpurun_out/sanitize_$tool.log | tail -5
done
