cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tg.py -x -q 2>&1 | grep -E "^E |passed|failed|Error" | head -20
DPG_TG_CK=4 DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=2 timeout 120 python tools/tg_trace_step.py 2>&1 | head -30
for v in 1 4; do
DPG_TG_CK=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ck$v.csv python tools/prof_step.py > /dev/null 2>&1
echo "== ck $v"; python tools/ncu_stages.py gpurun_out/ck$v.csv gpurun_out/stages_cifar_b512.json | grep -E "fwd|dgrad"
done
for v in 1 4; do
DPG_TG_CK=$v timeout 300 python bench.py --steps 300 > gpurun_out/bck_$v.json 2>gpurun_out/bck_$v.err; echo "rc $?"; tail -2 gpurun_out/bck_$v.err; python -c "
import json;d=json.load(open('gpurun_out/bck_$v.json'));print('ck=$v',round(d['ms_per_step'],4))"
done
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -4
