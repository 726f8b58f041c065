# GPU evidence pass: tests, smoke, bench (both arms), launch list, one ncu --set full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv > gpurun_out/launch_table.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_full python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
cat gpurun_out/bench.json; echo; cat gpurun_out/bench_ref.json
