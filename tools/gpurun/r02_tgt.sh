cd $GRAFT_REPO_ROOT
timeout 300 python tools/tg_time.py 2>&1 | tail -8
