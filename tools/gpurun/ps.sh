cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench10.json 2> gpurun_out/bench10.err; tail -2 gpurun_out/bench10.err
DPG_RS=0 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench10_tc.json 2>&1
python - <<'PY'
import json
a=json.load(open('gpurun_out/bench10.json')); b=json.load(open('gpurun_out/bench10_tc.json'))
print("ps ms/step", a["ms_per_step"], "value", a["value"], " tc ms/step", b["ms_per_step"])
sa=a["roofline"]["stages_ms"]; sb=b["roofline"]["stages_ms"]
for k in sorted(set(sa)|set(sb), key=lambda k:-max(sa.get(k,0),sb.get(k,0))):
    print(f"{k:22s} ps {sa.get(k,0)*1000:8.1f} us   tc {sb.get(k,0)*1000:8.1f} us")
PY
