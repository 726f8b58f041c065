cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none -k regex:persist -c 2 -o gpurun_out/persist python bench.py --workload mnist_b64 --steps 3 --warmup 3 > gpurun_out/persist_ncu.log 2>&1
tail -2 gpurun_out/persist_ncu.log
ncu -i gpurun_out/persist.ncu-rep --page details --launch-skip 1 --launch-count 1 2>/dev/null | grep -E "Duration|Grid Size|Block Size|Registers|Achieved Occupancy|Theoretical Occupancy|Dynamic Shared|Issue Slots|Executed Ipc" | head -20
