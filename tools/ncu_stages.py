"""Attribute an ncu capture of tools/prof_step.py to the step's stages.

    python tools/ncu_stages.py REPORT.ncu-rep|RAW.csv STAGES.json [OUT.json]

Kernels are matched to stages in launch order (prof_step.py runs the profiled step on one stream
and writes the stage sequence with its kernel counts). Per stage: ncu time (cold-cache,
serialised), DRAM bytes read + written (dram__bytes_read.sum + dram__bytes_write.sum) and the
algorithmic bytes the stage claims, so traffic / algorithmic shows wasted re-reads.
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}


def rows_of(path):
    if path.endswith(".csv"):
        text = open(path).read()
    else:
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                               "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                              check=True, capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(text)) if len(r) > 3]
    h = rows[0]
    if "Metric Name" in h:  # `ncu --csv --metrics ...` log: one row per (kernel, metric)
        ki, mi, ui, vi, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit",
                                                   "Metric Value", "ID"))
        per = {}
        for r in rows[1:]:
            d = per.setdefault(int(r[ii]), {"kernel": r[ki], "us": 0.0, "dram_bytes": 0.0})
            v = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
            if r[mi] == "gpu__time_duration.sum":
                d["us"] = v
            elif r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                d["dram_bytes"] += v
        return [per[i] for i in sorted(per)]
    units = rows[1]
    out = []
    for r in rows[2:]:
        def val(name):
            i = h.index(name)
            return float(r[i].replace(",", "")) * UNITS.get(units[i], 1.0)
        out.append({"kernel": r[h.index("Kernel Name")], "us": val("gpu__time_duration.sum"),
                    "dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum")})
    return out


def main(rep, stages_path, out_path=None):
    ks = rows_of(rep)
    stages = json.load(open(stages_path))
    if sum(s["kernels"] for s in stages) != len(ks):
        sys.exit(f"{len(ks)} kernels in the capture, {sum(s['kernels'] for s in stages)} in the stages")
    res, i = {}, 0
    for s in stages:
        part = ks[i:i + s["kernels"]]
        i += s["kernels"]
        res[s["stage"]] = {"ncu_us": sum(k["us"] for k in part),
                           "traffic": sum(k["dram_bytes"] for k in part),
                           "algorithmic_bytes": s["bytes"],
                           "kernels": [k["kernel"].split("(")[0] for k in part]}
    for k, v in res.items():
        print(f"{k:22s} {v['ncu_us']:8.2f} us  traffic {v['traffic'] / 1e6:8.2f} MB  "
              f"algorithmic {v['algorithmic_bytes'] / 1e6:8.2f} MB")
    if out_path:
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
