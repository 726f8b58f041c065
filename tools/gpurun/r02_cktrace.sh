cd $GRAFT_REPO_ROOT
for c in 0 100; do
DPG_TG_RESB=1 DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=5 DPG_TG_TRACE_CTA=$c timeout 120 python tools/tg_trace_step.py 2>&1 | tail -46
done
