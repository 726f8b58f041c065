cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/tg_trace_lin.py > /dev/null 2>&1; echo "plain rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tg_kernel -c 1 -o gpurun_out/lin_rule_full python tools/tg_trace_lin.py > gpurun_out/lin_ncu_full.log 2>&1; echo "ncu rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tg_kernel --launch-skip 1 -c 1 -o gpurun_out/lin_csum_full python tools/tg_trace_lin.py > gpurun_out/lin_ncu_full2.log 2>&1; echo "ncu2 rc $?"
