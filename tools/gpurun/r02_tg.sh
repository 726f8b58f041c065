cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tg.py -q 2>&1 | grep -E "^E |passed|failed" | head -20
