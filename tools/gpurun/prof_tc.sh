cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k regex:tc_gemm -c 20 -o gpurun_out/tc_all python tools/prof_step.py > gpurun_out/tc_all.log 2>&1
tail -2 gpurun_out/tc_all.log
