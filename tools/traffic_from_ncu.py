"""profiles/jcg_traffic.json from steady-state ncu --set full captures of K1 + K2 (one launch each):
DRAM bytes (read + write) per CG iteration, and the algorithmic bytes for comparison.
  python tools/traffic_from_ncu.py c4=gpurun_out/p_const.ncu-rep c3=gpurun_out/p_elem.ncu-rep"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALG = {"c4": (64, 511 ** 3), "c3": (80, 255 * 255 * 256)}   # bytes per unknown, free unknowns


def dram(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = []
    for d in data:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(d[i]) * scale[units[i]]
        t = float(d[hdr.index("gpu__time_duration.sum")]) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}[
            units[hdr.index("gpu__time_duration.sum")]]
        res.append({"kernel": d[hdr.index("Kernel Name")][:60], "dram_bytes": b, "seconds": t})
    return res


def main():
    out = {"note": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one steady-state K1 and one K2 "
                   "launch from ncu --set full (cold cache, serialised); algorithmic = bytes/unknown x free unknowns"}
    for arg in sys.argv[1:]:
        cfg, path = arg.split("=")
        ks = dram(path)
        bpu, nf = ALG[cfg]
        # 4 launches = K1, K2 with x, K1, K2 without x (deferred x update): two iterations
        tot = sum(k["dram_bytes"] for k in ks) / (len(ks) // 2)
        out[cfg] = {"bytes_per_iteration_k1_k2": tot, "algorithmic_bytes": bpu * nf,
                    "ratio": tot / (bpu * nf), "launches": ks, "source": os.path.basename(path)}
        if cfg == "c4" and len(ks) == 4:
            out[cfg]["moved_bytes_deferred_x"] = 60 * nf
            out[cfg]["ratio_to_moved"] = tot / (60 * nf)
    json.dump(out, open(os.path.join(ROOT, "profiles", "jcg_traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
