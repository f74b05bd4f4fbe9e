"""C4 512^3 lifted right-hand side b and ||b|| through level_rhs, saved to an .npy (A/B of library variants)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402

if os.environ.get("ECMG_LIB_PATH"):
    ecmg.LIB_PATH = os.environ["ECMG_LIB_PATH"]
g = Grid(4, 8, PROB["C4"])
b = g.new_vec(7)
nb = g.level_rhs(7, b)
np.save(sys.argv[1], b.cpu().numpy())
print("norm_b", repr(nb))
