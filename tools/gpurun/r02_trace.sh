cd $GRAFT_REPO_ROOT
for e in trace exp2 exp4 exp8; do echo "== $e"; DPG_LIB=libdpg_$e.so DPG_TG_TRACE_AT=0 timeout 120 python tools/tg_trace_step.py 2>&1 | grep -A1 "tile 0"; done
