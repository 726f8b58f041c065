# Iteration pass: GPU tests, bench (no CPU baseline), launch list + per-stage DRAM traffic.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -2 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/ncu_stages.py gpurun_out/launches.csv gpurun_out/stages_cifar_b512.json gpurun_out/ncu_traffic_cifar_b512.json
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms/step', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'], 'clocks', d['clocks'])"
