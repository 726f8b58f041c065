cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ps_conv_kernel -c 4 -o gpurun_out/ps_gs python tools/prof_step.py > gpurun_out/ps_gs.log 2>&1
tail -3 gpurun_out/ps_gs.log
