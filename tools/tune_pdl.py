"""Per-level JCG solve time of a full ecmg_run (C3, C4) with programmatic dependent launch on / off."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402


def main():
    for name, pid, levels, eps in (("c3", PROB["C3"], 7, 1e-10), ("c4", PROB["C4"], 8, 1e-9)):
        g = Grid(4, levels, pid)
        shape, nodes = g.shape(levels - 1)
        u = torch.empty(nodes, dtype=torch.float64, device="cuda")
        for pdl in (0, 1, 0, 1):
            g.set_option(ecmg.OPT_PDL, pdl)
            g.run(eps, u)
            best = None
            for _ in range(3):
                st, stats = g.run(eps, u)
                sol = [s["ms_solve"] for s in stats]
                if best is None or sum(sol) < sum(best):
                    best = sol
            print(json.dumps(dict(cfg=name, pdl=pdl, solve_ms=[round(v, 3) for v in best], total=round(sum(best), 3))),
                  flush=True)


if __name__ == "__main__":
    main()
