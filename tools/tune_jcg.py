"""Sweep the z-chunk size (planes per CTA) of the fixed-iteration fine-grid JCG benchmark (C4 512^3)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402


def main():
    g = Grid(4, 8, PROB["C4"])
    shape, nodes = g.shape(7)
    x0 = torch.from_numpy(synth.random_nodal(14, shape, (1, 1, 1), tuple(v - 1 for v in shape))).cuda()
    xb = x0.clone()
    out = []
    for kv in (1, 0):
        g.set_option(ecmg.OPT_KERNEL, kv)
        for zc in [int(a) for a in (sys.argv[1:] or [0, 511, 256, 171, 128, 86, 64, 43, 32, 16])]:
            g.set_option(ecmg.OPT_ZCHUNK, zc)
            g.solve_level(7, 0.0, 3, xb)
            best = 1e30
            for _ in range(3):
                xb.copy_(x0)
                g.solve_level(7, 0.0, 30, xb)
                ms, it, nf = g.last_jcg_timing()
                best = min(best, ms / it)
            gbs = 64 * nf / (best / 1e3) / 1e9
            out.append(dict(kernel=kv, zc=zc, ms_per_iter=best, gbs=gbs))
            print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
