cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -40 gpurun_out/pytest_gpu.log
