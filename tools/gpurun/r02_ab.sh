cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { # name env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 400 > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python -c "
import json;d=json.load(open('gpurun_out/ab_$name.json'));print('$name',round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
run old DPG_LIB=libdpg_old.so
run new_ck1_cs0 DPG_TG_CK=1 DPG_TG_CSUM=0
run new_ck1_cs1 DPG_TG_CK=1 DPG_TG_CSUM=1
run new_ck2_cs0 DPG_TG_CK=2 DPG_TG_CSUM=0
run new_ck4_cs0 DPG_TG_CK=4 DPG_TG_CSUM=0
run old_cs0 DPG_LIB=libdpg_old.so DPG_TG_CSUM=0
done
