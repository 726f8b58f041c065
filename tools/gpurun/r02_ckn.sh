cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 1 4; do
DPG_TG_CK=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ck$v.csv python tools/prof_step.py > /dev/null 2>&1
echo "== ck $v"; python tools/ncu_stages.py gpurun_out/ck$v.csv gpurun_out/stages_cifar_b512.json | grep -E "fwd|dgrad|csum"
done
