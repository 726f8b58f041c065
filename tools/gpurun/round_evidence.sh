# GPU evidence pass: tests, smoke, bench (both arms), launch list + per-stage traffic, ncu --set full.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/ncu_stages.py gpurun_out/launches.csv gpurun_out/stages_cifar_b512.json gpurun_out/ncu_traffic_cifar_b512.json > gpurun_out/launch_table.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_full python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
cat gpurun_out/launch_table.txt
