cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DIAG_ISOLATE=only timeout 300 python tools/diag_parity.py cifar_b4096 4096 1.48 > gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -rf > gpurun_out/pytest_full.log 2>&1; echo "pytest rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_full.log | head -20
