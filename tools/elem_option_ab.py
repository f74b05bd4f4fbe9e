"""Element-operator iteration (C5 1024^3 by default; argv: levels, C3 | C5, option) with an option off and on,
interleaved: BETA_FLY (beta formed on the fly from the per-axis tables, 64 instead of 80 B/unknown) or XDEFER
(the deferred x update, 76 B). 20 fixed iterations from x0 = 0, best of 3 each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 9
cfg = sys.argv[2] if len(sys.argv) > 2 else "C5"
g = Grid(4, levels, PROB[cfg], synth.c5_geometry(0) if cfg == "C5" else None)
k = levels - 1
_, nodes = g.shape(k)
x = torch.zeros(nodes, dtype=torch.float64, device="cuda")
opt = sys.argv[3] if len(sys.argv) > 3 else "BETA_FLY"
for fly in (0, 2, 0, 2) if opt == "XDEFER" else (0, 1, 0, 1):   # (XDEFER: 2 = also on the element operator)
    g.set_option(getattr(ecmg, "OPT_" + opt), fly)
    g.solve_level(k, 0.0, 2, x)
    best = 1e30
    for _ in range(3):
        x.zero_()
        g.solve_level(k, 0.0, 20, x)
        ms, it, nf = g.last_jcg_timing()
        best = min(best, ms / it)
    print(json.dumps(dict(cfg=cfg, n=4 << k, option=opt, value=fly, ms_per_iter=round(best, 4),
                          frac_at_80B=round(80 * nf / (best / 1e3) / 1e9 / 6553.6, 4))), flush=True)
