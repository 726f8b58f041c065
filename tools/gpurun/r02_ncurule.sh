cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DPG_TG_RULE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k regex:"ConvRuleT" -c 1 -o gpurun_out/rule_full python tools/prof_step.py > gpurun_out/ncu_rule.log 2>&1
tail -3 gpurun_out/ncu_rule.log
ls -la gpurun_out/rule_full.ncu-rep
