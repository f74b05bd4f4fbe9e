"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel (shares of the step)."""
import collections, csv, json, re, sys

def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        m = re.search(r'(k_\w+)(<[^>]*>)?', d['Kernel Name'])
        k = (m.group(1) + (m.group(2) or '')) if m else d['Kernel Name'][:40]
        scale = {'ns': 1e-6, 'nsecond': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}[d['Metric Unit']]
        agg[k][0] += 1
        agg[k][1] += float(d['Metric Value']) * scale
    tot = sum(v[1] for v in agg.values())
    return {"total_ms": tot, "kernels": {k: {"launches": v[0], "ms": round(v[1], 4), "share": round(v[1] / tot, 4)}
                                         for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}

if __name__ == "__main__":
    out = summarise(sys.argv[1])
    if len(sys.argv) > 2:
        out["what"] = sys.argv[2]
    print(json.dumps(out, indent=1))
