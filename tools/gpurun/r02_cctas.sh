cd $GRAFT_REPO_ROOT
for rep in 1 2; do for lib in libdpg.so libdpg_c2.so libdpg_c4.so libdpg_c6.so; do
  DPG_LIB=$lib timeout 300 python bench.py --steps 400 > gpurun_out/cc.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/cc.json'));r=d['roofline'];print('$lib',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in r['stages_ms'].items() if k.startswith('csum.conv')})"
done; done
