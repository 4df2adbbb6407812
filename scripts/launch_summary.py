"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

usage: python scripts/launch_summary.py launches.csv [--skip N]
Prints per kernel: launches, total ms, share, mean GB/s achieved from DRAM bytes.
"""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                     "Metric Unit")}
    launches = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        d = launches.setdefault(r[col["ID"]], {"name": r[col["Kernel Name"]]})
        v = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "byte": 1.0,
                 "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r[col["Metric Name"]]] = v * scale
    return list(launches.values())


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    ls = load(path)[skip:]
    agg = OrderedDict()
    for d in ls:
        a = agg.setdefault(d["name"][:70], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total ms | share | DRAM GB | GB/s |")
    print("|---|---|---|---|---|---|")
    for k, (n, ms, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% | {by / 1e9:.3f} | "
              f"{by / 1e9 / (ms / 1e3):.0f} |")


if __name__ == "__main__":
    main()
