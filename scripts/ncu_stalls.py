"""Top warp-stall reasons and hottest SASS lines of one kernel from
`ncu -i rep --page source --csv --print-source sass` output (first kernel).

usage: python scripts/ncu_stalls.py sass.csv [top]
"""
import csv
import sys


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    hi = next(i for i, r in enumerate(rows) if "Source" in r and any("Sampl" in c for c in r))
    hdr = rows[hi]
    data = []
    for r in rows[hi + 1:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(hdr):
            data.append(r)
    S = hdr.index("Warp Stall Sampling (All Samples)")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {h: sum(f(r[hdr.index(h)]) for r in data) for h in stalls}
    T = sum(tot.values()) or 1
    print(rows[0][1][:80], "samples", T)
    for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
        print(f"  {h:24s} {v / T:.3f}")
    for r in sorted(data, key=lambda r: -f(r[S]))[:top]:
        ex = sorted(((h, f(r[hdr.index(h)])) for h in stalls), key=lambda x: -x[1])[:2]
        print(f"  {r[1][:64]:64s} {f(r[S]):7.0f} {ex}")


if __name__ == "__main__":
    main()
