# usage: bash tools/gpurun/prof_k.sh <regex> <count> <name>
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k regex:$1 -c $2 -o gpurun_out/$3 python tools/prof_step.py > gpurun_out/$3.log 2>&1
tail -1 gpurun_out/$3.log
