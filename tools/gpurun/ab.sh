# A/B: bench stage times under two env settings. usage: bash tools/gpurun/ab.sh "ENV_A" "ENV_B"
cd $GRAFT_REPO_ROOT
env $1 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/ab_a.json 2>/dev/null
env $2 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/ab_b.json 2>/dev/null
python - <<'PY'
import json
a=json.load(open('gpurun_out/ab_a.json')); b=json.load(open('gpurun_out/ab_b.json'))
print("A ms/step", round(a['ms_per_step']*1000,1), " B ms/step", round(b['ms_per_step']*1000,1))
sa=a['roofline']['stages_ms']; sb=b['roofline']['stages_ms']
for k in sorted(set(sa)|set(sb), key=lambda k:-max(sa.get(k,0),sb.get(k,0)))[:24]: print(f"{k:22s} {sa.get(k,0)*1000:7.1f} {sb.get(k,0)*1000:7.1f}")
PY
