cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:conv_tc_kernel -s 1 -c 1 -o gpurun_out/cv_fwd2 python tools/prof_step.py > gpurun_out/ncu_cv.log 2>&1
tail -2 gpurun_out/ncu_cv.log
