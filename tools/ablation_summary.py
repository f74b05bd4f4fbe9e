"""Per-kernel time and DRAM bytes from an ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum launch list (one row per kernel and metric): totals per kernel and per iteration."""
import collections
import csv
import json
import re
import sys

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, iters, what):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: {"launches": 0, "s": 0.0, "dram_bytes": 0.0})
    for d in data:
        m = re.search(r"(k_\w+)(<[^>]*>)?", d["Kernel Name"])
        k = (m.group(1) + (m.group(2) or "")) if m else d["Kernel Name"][:40]
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[k]["launches"] += 1
            agg[k]["s"] += v
        else:
            agg[k]["dram_bytes"] += v
    tot_s = sum(a["s"] for a in agg.values())
    tot_b = sum(a["dram_bytes"] for a in agg.values())
    out = {"what": what, "iterations": iters, "total_ms": tot_s * 1e3, "total_dram_gb": tot_b / 1e9,
           "kernels": {k: {"launches": a["launches"], "ms": round(a["s"] * 1e3, 4), "dram_gb": round(a["dram_bytes"] / 1e9, 4)}
                       for k, a in sorted(agg.items(), key=lambda x: -x[1]["s"])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "")
