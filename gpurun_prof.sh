cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_full python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/step_full.ncu-rep
