"""Diagnostic: C4 512^3 right-hand side, GPU (level_rhs) vs oracle (Level.rhs): elementwise differences and
||b|| computed by each side, by numpy's pairwise sum and by math.fsum (exact rounding)."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as o
from paper_1506_02983_b200 import Grid

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 7
n = 4 << lev
g = Grid(4, lev + 1, o.C4)
b = g.new_vec(lev)
nb_g = g.level_rhs(lev, b)
bg = b.cpu().numpy()
g.close()
o.set_threads(o.max_threads())
t = time.time()
L = o.Level((n, n, n), o.C4)
bo, nb_o = L.rhs()
m, _ = L.dirichlet()
print(f"oracle level built in {time.time() - t:.1f} s")
fr = ~m
d = np.abs(bg - bo)
i = int(np.argmax(d))
nn = n + 1
print(f"n={n} nb_gpu={nb_g!r} nb_oracle={nb_o!r} rel={abs(nb_g - nb_o) / nb_o:.3e}")
print(f"max|db|={d.max():.3e} max|b|={np.abs(bo).max():.3e} at node {(i % nn, i // nn % nn, i // nn // nn)}"
      f" gpu {bg[i]!r} oracle {bo[i]!r}")
print(f"||db||_2={np.linalg.norm(bg[fr] - bo[fr]):.3e} dirichlet nonzero gpu {np.count_nonzero(bg[m])} oracle {np.count_nonzero(bo[m])}")
print(f"fsum gpu {math.sqrt(math.fsum((bg[fr] ** 2).tolist()))!r} fsum oracle {math.sqrt(math.fsum((bo[fr] ** 2).tolist()))!r}")
print(f"np pairwise gpu {math.sqrt(float(np.sum(bg[fr] ** 2)))!r} oracle {math.sqrt(float(np.sum(bo[fr] ** 2)))!r}")
top = np.argsort(d)[-10:]
for j in top:
    print((j % nn, j // nn % nn, j // nn // nn), bg[j], bo[j], d[j])
