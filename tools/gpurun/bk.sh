cd $GRAFT_REPO_ROOT
python bench.py --no-cpu-baseline > gpurun_out/bk16.json 2>/dev/null
DPG_LIB=libdpg_bk32.so python bench.py --no-cpu-baseline > gpurun_out/bk32.json 2>/dev/null
DPG_LIB=libdpg_bk32.so timeout 300 python -m pytest tests/test_gpu_step.py -x -q 2>&1 | tail -1
python - <<'PY'
import json
a=json.load(open('gpurun_out/bk16.json')); b=json.load(open('gpurun_out/bk32.json'))
print("bk16", a['ms_per_step'], "bk32", b['ms_per_step'])
sa=a['roofline']['stages_ms']; sb=b['roofline']['stages_ms']
for k in sorted(sa, key=lambda k:-sa[k])[:20]: print(f"{k:22s} {sa[k]*1000:7.1f} {sb.get(k,0)*1000:7.1f}")
PY
