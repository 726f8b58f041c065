cd $GRAFT_REPO_ROOT
( time python bench.py ) > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -3 gpurun_out/bench_full.err
( time python bench.py --impl reference ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/bench_ref.err
cat gpurun_out/bench_full.json; echo; cat gpurun_out/bench_ref.json
