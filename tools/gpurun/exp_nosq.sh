cd $GRAFT_REPO_ROOT
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e1.json 2>/dev/null
touch paper_2109_12298_b200/csrc/rows_conv.cu
make -C $GRAFT_REPO_ROOT/paper_2109_12298_b200/csrc -j8 EXTRA="-DDPG_EXPERIMENT_NOSQ" > /dev/null 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e2.json 2>/dev/null
python - <<'PY'
import json
a=json.load(open('gpurun_out/e1.json'))["roofline"]["stages_ms"]; b=json.load(open('gpurun_out/e2.json'))["roofline"]["stages_ms"]
for k in ["gs.conv2d[4]","gs.conv2d[6]"]: print(k, a[k]*1000, b[k]*1000)
PY
