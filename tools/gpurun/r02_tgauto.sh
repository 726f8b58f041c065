cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rf > gpurun_out/ta_t.log 2>&1; echo "gpu suite rc $?"; tail -3 gpurun_out/ta_t.log
for wl in mnist_b64 cifar_b512 cifar_poisson; do for i in 1 2; do timeout 300 python bench.py --workload $wl --steps 500 > gpurun_out/ta.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/ta.json'));print('$wl',round(d['value']),round(d['ms_per_step'],4))"; done; done
