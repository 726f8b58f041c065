cd $GRAFT_REPO_ROOT
for d in 0 1 2 3 4 7; do
  DPG_TC_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/dbg_$d.csv python tools/prof_step.py > /dev/null 2>&1
  echo "== dbg $d"; python tools/ncu_stages.py gpurun_out/dbg_$d.csv gpurun_out/stages_cifar_b512.json | grep -E "fwd.conv|gs.conv2d\[[02]\]|dgrad.conv|csum.conv"
done
DPG_TC_WS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/dbg_old.csv python tools/prof_step.py > /dev/null 2>&1
echo "== old"; python tools/ncu_stages.py gpurun_out/dbg_old.csv gpurun_out/stages_cifar_b512.json | grep -E "fwd.conv|gs.conv2d\[[02]\]|dgrad.conv|csum.conv"
