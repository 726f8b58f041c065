"""Per-stage DRAM traffic of cfg2 (linear_t64) from an ncu launch list of tools/tg_trace_lin.py.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
        python tools/tg_trace_lin.py > lin_launch.csv
    python tools/lin_traffic.py lin_launch.csv > profiles/ncu_traffic_linear_t64.json

tg_trace_lin.py calls the rule (tg_kernel LinRuleT, sq_reduce, gs_bias), then a torch RNG kernel,
then the clipped sum (tg_kernel LinCsumT, splitk_reduce4, gs_bias, weighted_sum_narrow): bench.py's
stages "gs.linear+bias" and "csum.linear+bias"."""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
k = {}
for r in rows:
    k.setdefault(int(r[0]), {"name": r[4]})[r[12]] = float(r[14].replace(",", ""))
ids = sorted(k)
stage = {"gs.linear+bias": [], "csum.linear+bias": []}
cur = "gs.linear+bias"
for i in ids:
    n = k[i]["name"]
    if "LinCsumT" in n:
        cur = "csum.linear+bias"
    if "at::" in n:  # the test's own RNG kernel between the two calls
        continue
    stage[cur].append(i)
out = {"_source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum, "
                  "tools/tg_trace_lin.py (b=256, T=64, d=r=512)"}
for sn, ii in stage.items():
    out[sn] = {"ncu_us": sum(k[i]["gpu__time_duration.sum"] for i in ii) / 1000.0,
               "traffic": sum(k[i]["dram__bytes_read.sum"] + k[i]["dram__bytes_write.sum"] for i in ii),
               "kernels": [k[i]["name"][:90] for i in ii]}
print(json.dumps(out, indent=1))
