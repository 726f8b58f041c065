cd $GRAFT_REPO_ROOT
for k in 5 6; do
DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=$k timeout 120 python tools/tg_trace_step.py 2>&1 | tail -22
done
