cd $GRAFT_REPO_ROOT
for lib in libdpg.so libdpg_s3.so libdpg_s2.so libdpg_g96.so libdpg.so; do
DPG_LIB=$lib timeout 300 python bench.py --steps 300 > gpurun_out/b_$lib.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b_$lib.json'));st=d['roofline']['stages_ms'];print('$lib',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'fwd' in k or 'dgrad' in k})"
done
