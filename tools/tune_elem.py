"""A/B timing of libecmg builds on the element path (C3 256^3 fixed-iteration JCG) and the constant path
(C4 512^3). Usage: python tools/tune_elem.py lib1.so lib2.so ...  -- each build is timed in its own process
(ecmg.LIB_PATH is pointed at it before the library is loaded; tuning only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(path, cfg, zcs=(0,)):
    sys.path.insert(0, ROOT)
    import torch
    import synth
    from paper_1506_02983_b200 import Grid, PROB, ecmg
    ecmg.LIB_PATH = os.path.abspath(path)
    pid, n0, levels = {"c3": (PROB["C3"], 4, 7), "c4": (PROB["C4"], 4, 8), "c4_256": (PROB["C4"], 4, 7),
                       "c5": (PROB["C5"], 4, 9), "c3_128": (PROB["C3"], 4, 6)}[cfg]
    g = Grid(n0, levels, pid, synth.c5_geometry(0) if cfg == "c5" else None)
    k = levels - 1
    shape, nodes = g.shape(k)
    x0 = torch.from_numpy(synth.random_nodal(14, shape, (1, 1, 1), tuple(v - 1 for v in shape))).cuda()
    xb = x0.clone()
    for zc in zcs:
        g.set_option(ecmg.OPT_ZCHUNK, zc)
        g.solve_level(k, 0.0, 3, xb)
        best = 1e30
        for _ in range(3):
            xb.copy_(x0)
            g.solve_level(k, 0.0, 40, xb)
            ms, it, nf = g.last_jcg_timing()
            best = min(best, ms / it)
        bpu = 80 if cfg in ("c3", "c5", "c3_128") else 64
        print(json.dumps(dict(lib=os.path.basename(path), cfg=cfg, zc=zc, ms_per_iter=round(best, 5),
                              frac=round(bpu * nf / (best / 1e3) / 1e9 / 6553.6, 4))), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        one(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "--zc":   # --zc lib cfg zc1 zc2 ...
        one(sys.argv[2], sys.argv[3], [int(v) for v in sys.argv[4:]])
    else:
        for p in sys.argv[1:]:
            for cfg in ("c3", "c4"):
                subprocess.run([sys.executable, __file__, "--one", p, cfg], timeout=300)
