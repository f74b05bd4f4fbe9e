import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1506_02983_b200 import Grid, PROB, ecmg
g = Grid(4, 3, PROB["C1"])
for kv in (0, 1):
    g.set_option(ecmg.OPT_KERNEL, kv)
    p = torch.rand(g.shape(2)[1], dtype=torch.float64, device="cuda")
    q = torch.zeros_like(p)
    st = ecmg.apply_operator(g.h, 2, p, q)
    torch.cuda.synchronize()
    print("kernel", kv, "apply status", st, float(q.abs().max()))
