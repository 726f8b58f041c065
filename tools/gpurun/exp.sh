# tc kernel cost breakdown: ncu launch times with gathers / stores / MMAs skipped (wrong results)
cd $GRAFT_REPO_ROOT
for e in 0 1 2 4 7; do
  lib=libdpg.so; [ $e != 0 ] && lib=libdpg_exp$e.so
  DPG_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/exp_$e.csv python tools/prof_step.py > /dev/null 2>&1
  python tools/ncu_stages.py gpurun_out/exp_$e.csv gpurun_out/stages_cifar_b512.json > gpurun_out/exp_$e.txt
done
python - <<'PY'
import re
rows={}
for e in [0,1,2,4,7]:
    for line in open(f'gpurun_out/exp_{e}.txt'):
        m=re.match(r'(\S+)\s+([\d.]+) us', line)
        if m: rows.setdefault(m.group(1),{})[e]=float(m.group(2))
print(f"{'stage':22s} {'full':>7s} {'-gath':>7s} {'-store':>7s} {'-mma':>7s} {'-all':>7s}")
for k,v in rows.items():
    if any(s in k for s in ('fwd.conv','dgrad.conv','gs.conv2d[2]','csum.conv')):
        print(f"{k:22s} " + " ".join(f"{v.get(e,0):7.1f}" for e in [0,1,2,4,7]))
PY
