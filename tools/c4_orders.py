"""C4 errors against the exact solution (L_inf and RMS over all nodes) of u_h and u~_h at 128^3..512^3 for
two tolerances (diagnostic for the full-size property test)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB  # noqa: E402


def exact(n):
    z, y, x = torch.meshgrid(*[torch.arange(n + 1, dtype=torch.float64, device="cuda") / n for _ in range(3)], indexing="ij")
    return ((x * x + y * y + z * z) ** 0.75).reshape(-1)


for eps in (1e-9, 1e-12):
    for lv in (6, 7, 8):
        g = Grid(4, lv, PROB["C4"])
        u, ut = g.new_vec(lv - 1), g.new_vec(lv - 1)
        st, stats = g.run(eps, u, ut)
        ue = exact(4 << (lv - 1))
        e, et = u - ue, ut - ue
        print(json.dumps(dict(eps=eps, n=4 << (lv - 1), st=st, its=[s["iterations"] for s in stats],
                              u_inf=float(e.abs().max()), u_rms=float(e.pow(2).mean().sqrt()),
                              ut_inf=float(et.abs().max()), ut_rms=float(et.pow(2).mean().sqrt()))), flush=True)
        del u, ut, ue, e, et
        g.close()
        torch.cuda.empty_cache()
