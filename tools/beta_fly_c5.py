"""C5 1024^3 element iteration with beta read from the array (80 B/unknown) vs formed on the fly from the
per-axis tables (64 B/unknown; ECMG_OPT_BETA_FLY) -- or any other 0/1 option named as argv[3], e.g. XDEFER: 20 fixed iterations from x0 = 0, best of 3 each."""
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
for fly in (0, 1, 0, 1):
    g.set_option(getattr(ecmg, "OPT_" + (sys.argv[3] if len(sys.argv) > 3 else "BETA_FLY")), fly)
    g.solve_level(k, 0.0, 2, x)
    best = 1e30
    for _ in range(3):
        x.zero_()
        g.solve_level(k, 0.0, 20, x)
        ms, it, nf = g.last_jcg_timing()
        best = min(best, ms / it)
    print(json.dumps(dict(cfg=cfg, n=4 << k, option=(sys.argv[3] if len(sys.argv) > 3 else "BETA_FLY"), value=fly, ms_per_iter=round(best, 4),
                          frac_at_80B=round(80 * nf / (best / 1e3) / 1e9 / 6553.6, 4))), flush=True)
