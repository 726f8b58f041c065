cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/tg_trace_lin.py > /dev/null 2>&1; echo "plain rc $?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/tg_trace_lin.py > gpurun_out/lin_launch.csv 2>&1; echo "ncu rc $?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/lin_launch.csv')) if len(r)>10 and r[0].isdigit()]
from collections import OrderedDict
k=OrderedDict()
for r in rows:
    k.setdefault((r[0],r[4][:70]),{})[r[12]]=r[14]
for (i,n),m in k.items(): print(i,n,m)
PY
