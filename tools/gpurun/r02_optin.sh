cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "alternate_paths" 2>&1 | tail -3
DPG_TG_RULE=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3" 2>&1 | tail -3
