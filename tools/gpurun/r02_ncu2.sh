cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"tg_kernel" -c 2 -o gpurun_out/tg2 python tools/prof_step.py > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
