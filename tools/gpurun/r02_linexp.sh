cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in "" exp1 exp2; do
  lib=libdpg${e:+_$e}.so
  DPG_LIB=$lib timeout 300 python bench.py --workload linear_t64 --steps 50 > gpurun_out/linexp_$e.json 2> gpurun_out/linexp_$e.err; echo "$lib rc $?"
  python -c "
import json;d=json.load(open('gpurun_out/linexp_$e.json'));r=d['roofline'];print(d['ms_per_step'],r.get('stages_ms'))"
done
