cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__occupancy_limit_shared_mem --clock-control none --profile-from-start off --csv --log-file gpurun_out/kl2_cv.csv python tools/prof_step.py > /dev/null 2>&1
DPG_CV=0 timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__occupancy_limit_shared_mem --clock-control none --profile-from-start off --csv --log-file gpurun_out/kl2_tc.csv python tools/prof_step.py > /dev/null 2>&1
ls -la gpurun_out/kl_*.csv
