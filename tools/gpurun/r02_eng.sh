cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg_linear.py -k engine -rf > gpurun_out/eng.log 2>&1; echo "engine rc $?"; tail -15 gpurun_out/eng.log
DPG_TG_LIN=0 timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_tg_linear.py -k engine -rf > gpurun_out/eng0.log 2>&1; echo "engine TG_LIN=0 rc $?"; tail -3 gpurun_out/eng0.log
timeout 300 python bench.py --workload linear_t64 > gpurun_out/cfg_linear_t64.json 2> /dev/null; echo "cfg2 rc $?"
