cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base function -k regex:^tk_ -o gpurun_out/tk python tools/prof_step.py > gpurun_out/tk.log 2>&1
tail -2 gpurun_out/tk.log
