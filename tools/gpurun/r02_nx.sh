cd $GRAFT_REPO_ROOT
for lib in libdpg.so libdpg_nx.so libdpg.so libdpg_nx.so; do
  DPG_LIB=$lib timeout 300 python bench.py --workload linear_t64 --steps 100 > gpurun_out/nx.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/nx.json'));r=d['roofline'];print('$lib lin',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items()})"
done
