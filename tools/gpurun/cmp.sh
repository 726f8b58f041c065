cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -2 gpurun_out/bench9.err
DPG_CV=0 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench9_tc.json 2>&1
python - <<'PY'
import json
a=json.load(open('gpurun_out/bench9.json')); b=json.load(open('gpurun_out/bench9_tc.json'))
print("cv ms/step", a["ms_per_step"], "value", a["value"], " tc ms/step", b["ms_per_step"])
sa=a["roofline"]["stages_ms"]; sb=b["roofline"]["stages_ms"]
for k in sorted(sa, key=lambda k:-sa[k]):
    print(f"{k:22s} cv {sa[k]*1000:8.1f} us   tc {sb.get(k,0)*1000:8.1f} us")
PY
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__occupancy_limit_shared_mem --clock-control none --profile-from-start off --csv --log-file gpurun_out/kl2_cv.csv python tools/prof_step.py > /dev/null 2>&1
DPG_CV=0 timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__occupancy_limit_shared_mem --clock-control none --profile-from-start off --csv --log-file gpurun_out/kl2_tc.csv python tools/prof_step.py > /dev/null 2>&1
ls -la gpurun_out/kl_*.csv
