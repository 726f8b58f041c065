"""Per-stage summary of an `ncu --set full` capture of tools/prof_step.py (one eager step).

    python tools/ncu_summary.py REPORT.ncu-rep STAGES.json > profiles/<round>_ncu_step.md

Columns: ncu duration (cold cache, serialised replay), DRAM bytes (read + write), DRAM GB/s, SM
throughput %, tensor pipe active %, issue active %, warps active %, registers, top warp stalls.
Kernels are attributed to stages in launch order (prof_step.py runs the profiled step on one
stream and records each stage's kernel count)."""
import csv
import io
import json
import subprocess
import sys

M = {
    "us": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "sm": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tc": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "iss": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1,
        "msecond": 1e3, "ms": 1e3}


def main(rep, stages_path):
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                          text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h, units = rows[0], rows[1]
    stall = [i for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not c.endswith("_not_issued")]
    ks = []
    for r in rows[2:]:
        d = {"name": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, c in M.items():
            i = h.index(c)
            try:
                d[k] = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
            except ValueError:
                d[k] = 0.0
        st = sorted(((float(r[i].replace(",", "") or 0), h[i][len("smsp__pcsamp_warps_issue_stalled_"):])
                     for i in stall), reverse=True)
        tot = sum(v for v, _ in st) or 1.0
        d["stalls"] = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:3])
        ks.append(d)
    stages = json.load(open(stages_path))
    print("| stage | kernel | ncu us | DRAM MB | DRAM GB/s | SM % | tensor % | issue % | warps % | regs | grid | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    i = 0
    tot_us = 0.0
    for s in stages:
        for k in ks[i:i + s["kernels"]]:
            mb = (k["rd"] + k["wr"]) / 1e6
            tot_us += k["us"]
            print(f"| {s['stage']} | {k['name'][:40]} | {k['us']:.1f} | {mb:.1f} | {mb / k['us'] * 1e3 if k['us'] else 0:.0f} | "
                  f"{k['sm']:.0f} | {k['tc']:.1f} | {k['iss']:.0f} | {k['warps']:.0f} | {k['regs']:.0f} | {k['grid']:.0f} | {k['stalls']} |")
        i += s["kernels"]
    print(f"\n{len(ks)} kernels, {tot_us:.1f} us serialised (cold-cache ncu replay; the graph overlaps branches)")


if __name__ == "__main__":
    main(*sys.argv[1:])
