# Every BASELINE config through bench.py (1 GPU): our arm + the reference CPU arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cifar_b512 linear_t64 mnist_b64 embed_b512 cifar_b4096; do
  timeout 600 python bench.py --workload $w > gpurun_out/cfg_$w.json 2> gpurun_out/cfg_$w.err; echo "$w rc $?"; tail -2 gpurun_out/cfg_$w.err
  timeout 600 python bench.py --workload $w --impl reference --steps 5 --warmup 1 > gpurun_out/cfgref_$w.json 2> gpurun_out/cfgref_$w.err; echo "$w ref rc $?"
done
python - <<'PY'
import json
for w in ["cifar_b512","linear_t64","mnist_b64","embed_b512","cifar_b4096"]:
    try:
        d=json.load(open(f"gpurun_out/cfg_{w}.json")); r=json.load(open(f"gpurun_out/cfgref_{w}.json"))
        print(f"{w:12s} {d['value']:12.0f} samples/s  {d['ms_per_step']:8.3f} ms  e2e {d['e2e']['value']:12.0f}  frac {d['roofline']['frac']:.3f} ({d['roofline']['kernel']})  cpu {r['value']:10.1f}")
    except Exception as e:
        print(w, "ERR", e)
PY
