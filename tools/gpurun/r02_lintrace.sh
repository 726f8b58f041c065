cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in 0 1; do DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=$k timeout 120 python tools/tg_trace_lin.py > gpurun_out/lintrace_$k.txt 2>&1; echo "trace $k rc $?"; head -60 gpurun_out/lintrace_$k.txt; done
timeout 300 ncu --kernel-name regex:tg_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum --clock-control none --csv python tools/tg_trace_lin.py > gpurun_out/lin_ncu.csv 2>&1; echo "ncu rc $?"; grep -v "^==" gpurun_out/lin_ncu.csv | tail -20
