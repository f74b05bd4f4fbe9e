"""z-chunk sweep of the fixed-iteration JCG on intermediate levels (64^3, 128^3) of C4 and C3."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402


def main():
    for name, pid in (("c4", PROB["C4"]), ("c3", PROB["C3"])):
        g = Grid(4, 6, pid)
        g.set_option(ecmg.OPT_PERSISTENT, 0)
        for k in (4, 5):
            shape, nodes = g.shape(k)
            x0 = torch.from_numpy(synth.random_nodal(14, shape, (1, 1, 1), tuple(v - 1 for v in shape))).cuda()
            xb = x0.clone()
            for zc in (0, 3, 4, 6, 8, 11, 16, 22, 32, 43, 64, 128):
                g.set_option(ecmg.OPT_ZCHUNK, zc)
                g.solve_level(k, 0.0, 3, xb)
                best = 1e30
                for _ in range(3):
                    xb.copy_(x0)
                    g.solve_level(k, 0.0, 50, xb)
                    ms, it, nf = g.last_jcg_timing()
                    best = min(best, ms / it)
                print(json.dumps(dict(cfg=name, level=k, n=shape[0] - 1, zc=zc, us_per_iter=round(best * 1e3, 2))), flush=True)


if __name__ == "__main__":
    main()
