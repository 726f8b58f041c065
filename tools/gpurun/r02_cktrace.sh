cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tg.py -x -q 2>&1 | grep -E "^E |passed|failed|Error" | head -20
for c in 0 1; do
DPG_TG_CK=4 DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=2 DPG_TG_TRACE_CTA=$c timeout 120 python tools/tg_trace_step.py 2>&1 | head -30
done
for v in 1 4; do
DPG_TG_CK=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ck$v.csv python tools/prof_step.py > /dev/null 2>&1
echo "== ck $v"; python tools/ncu_stages.py gpurun_out/ck$v.csv gpurun_out/stages_cifar_b512.json | grep -E "fwd|dgrad"
done
