cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"conv_fwd_thin" -c 1 -o gpurun_out/thin_full python tools/prof_step.py > gpurun_out/ncu_thin.log 2>&1
tail -2 gpurun_out/ncu_thin.log
