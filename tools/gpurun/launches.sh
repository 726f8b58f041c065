# per-kernel device time of one eager CIFAR step (launch list, ncu single pass per kernel)
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv
