cd $GRAFT_REPO_ROOT
for k in 0 1 2 3 4 5 6 7; do
DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=$k timeout 120 python tools/tg_trace_step.py 2>&1 | head -40
done
