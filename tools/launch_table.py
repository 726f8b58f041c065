"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel) as a table."""
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    tot = 0.0
    out = []
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        t = float(r[vi].replace(",", "")) / 1000.0
        tot += t
        out.append((t, r[ki]))
    for t, k in out:
        print(f"{t:8.2f} us  {k[:100]}")
    print(f"total {tot:.1f} us over {len(out)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
