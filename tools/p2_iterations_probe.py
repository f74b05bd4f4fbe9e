import sys; sys.path.insert(0, '.')
import torch
from paper_1506_02983_b200 import Grid
import oracle as o
for var in (1, 0):
    g = Grid((10, 4, 5), 5, o.P2, exp_variant=var)
    u = g.new_vec(4)
    st, stats = g.run(1e-12, u)
    print("variant", var, "iters", [s["iterations"] for s in stats], "rre", ["%.2e" % s["rel_res_true"] for s in stats])
