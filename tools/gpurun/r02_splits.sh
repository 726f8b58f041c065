cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 400 > gpurun_out/bsp.json 2>gpurun_out/bsp.err; python -c "
import json;d=json.load(open('gpurun_out/bsp.json'));st=d['roofline']['stages_ms'];print('$name',round(d['ms_per_step'],4),{k:round(v*1e3,1) for k,v in st.items() if 'csum' in k})"; }
run default
run small888 DPG_CSUM_CTAS_SMALLP=888
run all592 DPG_CSUM_CTAS=592
run all888 DPG_CSUM_CTAS=888
