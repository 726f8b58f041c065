cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" 1 L2 L4 L6 L2,4 L4,6; do
  DPG_TG_CSUM=$v timeout 300 python bench.py --steps 300 > gpurun_out/csumab.json 2> gpurun_out/csumab.err
  python -c "
import json;d=json.load(open('gpurun_out/csumab.json'));r=d['roofline'];s=r['stages_ms'];print('DPG_TG_CSUM=$v',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in s.items() if k.startswith('csum')})"
done
