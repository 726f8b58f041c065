cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_persist.py -q -x 2>&1 | tail -5
DPG_LIB=libdpg_ptrace.so timeout 120 python tools/persist_trace.py
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_norm.py tests/test_golden.py -q 2>&1 | tail -3
timeout 300 python bench.py --workload mnist_b64 > gpurun_out/cfg_mnist.json 2> gpurun_out/cfg_mnist.err; echo "rc $?"; tail -2 gpurun_out/cfg_mnist.err; python -c "
import json;d=json.load(open('gpurun_out/cfg_mnist.json'));print(d['value'],d['ms_per_step'],d.get('gpu_launches'))"
