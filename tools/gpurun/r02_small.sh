cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rules.py tests/test_gpu_step.py tests/test_gpu_tg.py > gpurun_out/small_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/small_tests.log
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fullsize.py -k "cfg2 or cfg3_cifar_b512" > gpurun_out/small_full.log 2>&1; echo "full rc $?"; tail -3 gpurun_out/small_full.log
timeout 120 python tools/tg_trace_lin.py > /dev/null 2>&1; echo "plain rc $?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/tg_trace_lin.py > gpurun_out/lin_launch.csv 2>&1; echo "ncu rc $?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/lin_launch.csv')) if len(r)>10 and r[0].isdigit()]
from collections import OrderedDict
k=OrderedDict()
for r in rows:
    k.setdefault((r[0],r[4][:60]),{})[r[12]]=r[14]
for (i,n),m in k.items(): print(i,n,m.get('gpu__time_duration.sum'))
PY
timeout 300 python bench.py --workload linear_t64 > gpurun_out/lin_bench.json 2> gpurun_out/lin_bench.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/lin_bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('stages_ms'))"
timeout 300 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/c_bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['kernel'],r['frac'],r.get('stages_ms'))"
