"""A/B of ecmg_run options on C4 (4^3 -> 512^3, eps 1e-9): the settings alternate run by run, N runs each,
median and quartiles of the CUDA-event TTS and of every level's solve time.
Usage: python tools/tts_ab.py N OPT=VAL[,OPT=VAL] OPT=VAL ...   (OPT: an ecmg.OPT_* name without the prefix;
every setting must name every option any setting changes)"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402

if os.environ.get("ECMG_LIB_PATH"):   # A/B of a variant build (tuning only)
    ecmg.LIB_PATH = os.environ["ECMG_LIB_PATH"]


def parse(spec):
    out = []
    for kv in spec.split(","):
        if kv:
            k, v = kv.split("=")
            out.append((getattr(ecmg, "OPT_" + k), int(v)))
    return out


def main():
    n = int(sys.argv[1])
    settings = [parse(s) for s in sys.argv[2:]] or [[]]
    cfg = os.environ.get("TTS_CFG", "c4")
    pid, L, eps = {"c4": ("C4", 8, 1e-9), "c3": ("C3", 7, 1e-10)}[cfg]
    g = Grid(4, L, PROB[pid])
    shape, nodes = g.shape(L - 1)
    u = torch.empty(nodes, dtype=torch.float64, device="cuda")
    ut = torch.empty(nodes, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    res = [[] for _ in settings]
    lv = [[] for _ in settings]
    for r in range(n + 2):
        for i, s in enumerate(settings):
            for o, v in s:
                g.set_option(o, v)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _, stats = g.run(eps, u, ut)
            e1.record(st)
            torch.cuda.synchronize()
            if r >= 2:
                res[i].append(e0.elapsed_time(e1))
                lv[i].append([(s_["ms_setup"], s_["ms_exp"], s_["ms_solve"], s_["ms_rich"]) for s_ in stats])
    for i, s in enumerate(sys.argv[2:] or ["default"]):
        q = statistics.quantiles(res[i], n=4)
        per = [[round(statistics.median(v[j] for v in x), 3) for j in range(4)] for x in zip(*lv[i])]
        print(json.dumps({"setting": s, "tts_median": round(statistics.median(res[i]), 3), "q1": round(q[0], 3),
                          "q3": round(q[2], 3), "per_level_median_setupwait_exp_solve_rich": per}), flush=True)


if __name__ == "__main__":
    main()
