"""Summarise an `ncu --set full` capture of the GEMM launches into
profiles/<name>.json (per-launch duration, DRAM bytes, tensor-pipe activity;
mean DRAM bytes per launch is what bench.py reports as roofline.traffic).

usage: python scripts/ncu_gemm_summary.py capture.ncu-rep out.json "<how it was captured>"
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1, "hz": 1, "Ghz": 1e9,
         "Mhz": 1e6, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def main():
    rep, out, how = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_col = hdr.index("Kernel Name")
    launches = []
    for r in data:
        d = {"kernel": r[name_col].split("(")[0]}
        for k, short in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                v = float(r[i].replace(",", ""))
                d[short] = v * SCALE.get(units[i], 1)
        launches.append(d)
    b = [l["dram_read"] + l["dram_write"] for l in launches if "dram_read" in l]
    res = {"source": how, "launches": launches,
           "mean_dram_bytes_per_gemm_launch": sum(b) / len(b) if b else None}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({"launches": len(launches), "mean_dram_bytes": res["mean_dram_bytes_per_gemm_launch"]}))


if __name__ == "__main__":
    main()
