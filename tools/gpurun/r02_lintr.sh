cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in 0; do DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=$k timeout 120 python tools/tg_trace_lin.py > gpurun_out/lintrace_$k.txt 2>&1; echo "trace $k rc $?"; grep tile gpurun_out/lintrace_$k.txt | head -8; done
