cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/ncu_stages.py gpurun_out/launches.csv gpurun_out/stages_cifar_b512.json gpurun_out/ncu_traffic_cifar_b512.json > gpurun_out/launch_table.txt 2>&1
cat gpurun_out/launch_table.txt | head -60
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"tg_kernel|im2col|prep_weights" -o gpurun_out/tg_full python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
