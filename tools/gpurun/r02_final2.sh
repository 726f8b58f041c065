# Round-2 re-entry evidence pass: full GPU suite, smoke, bench (both arms, every config), launch
# list, ncu step summary, timeline, the T > 1 linear kernels' launch list / ncu capture / traffic,
# a 2-rank protocol check (the compute sanitizer is closed on the GPU pool).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; head -c 300 gpurun_out/bench.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
for wl in mnist_b64 linear_t64 embed_b512 cifar_b4096 cifar_poisson; do timeout 600 python bench.py --workload $wl > gpurun_out/cfg_$wl.json 2> gpurun_out/cfg_$wl.err; echo "cfg $wl rc $?"; done
timeout 600 python bench.py --no-materialise > gpurun_out/cfg_cifar_b512_norms_only.json 2> gpurun_out/cfg_norms.err; echo "norms-only rc $?"
for wl in mnist_b64 linear_t64 embed_b512 cifar_b4096; do timeout 600 python bench.py --impl reference --workload $wl > gpurun_out/cfgref_$wl.json 2> gpurun_out/cfgref_$wl.err; echo "cfgref $wl rc $?"; done
timeout 300 python tools/graph_timeline.py > gpurun_out/timeline_cifar_b512.txt 2>&1; echo "timeline rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/ncu_stages.py gpurun_out/launches.csv gpurun_out/stages_cifar_b512.json gpurun_out/ncu_traffic_cifar_b512.json > gpurun_out/launch_table.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_full python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/tg_trace_lin.py > gpurun_out/lin_launch.csv 2>&1; echo "lin ncu rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tg_kernel -c 2 -o gpurun_out/lin_full python tools/tg_trace_lin.py > gpurun_out/lin_ncu_full.log 2>&1; echo "lin ncu full rc $?"
python tools/lin_traffic.py gpurun_out/lin_launch.csv > gpurun_out/ncu_traffic_linear_t64.json 2>&1; echo "lin traffic rc $?"
timeout 600 python bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench n2 (protocol check, both ranks on cuda:0) rc $?"; head -c 300 gpurun_out/bench_n2.json; echo
timeout 300 python bench.py --workload linear_t64 > gpurun_out/cfg_linear_t64_b.json 2> /dev/null; echo "cfg2 again rc $?"
