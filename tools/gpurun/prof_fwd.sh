cd $GRAFT_REPO_ROOT
DPG_PS=0 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k regex:ConvFwd -c 2 -o gpurun_out/tc_fwd python tools/prof_step.py > gpurun_out/tc_fwd.log 2>&1
DPG_PS=0 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k regex:ConvCsum -c 2 -o gpurun_out/tc_csum python tools/prof_step.py > gpurun_out/tc_csum.log 2>&1
tail -2 gpurun_out/tc_fwd.log
