"""Per-level JCG solve time of a full ecmg_run (C3 and C4) vs the persistent-kernel threshold
(ECMG_OPT_PERSISTENT = max free unknowns solved in one cooperative launch)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402


def main():
    pmaxs = [int(v) for v in sys.argv[1:]] or [0, 5000, 40000, 300000, 2200000]
    for name, pid, levels, eps in (("c3", PROB["C3"], 7, 1e-10), ("c4", PROB["C4"], 8, 1e-9)):
        g = Grid(4, levels, pid)
        shape, nodes = g.shape(levels - 1)
        u = torch.empty(nodes, dtype=torch.float64, device="cuda")
        for pm in pmaxs:
            g.set_option(ecmg.OPT_PERSISTENT, pm)
            g.run(eps, u)
            best = None
            for _ in range(3):
                st, stats = g.run(eps, u)
                sol = [s["ms_solve"] for s in stats]
                if best is None or sum(sol) < sum(best[0]):
                    best = (sol, [s["iterations"] for s in stats])
            print(json.dumps(dict(cfg=name, pmax=pm, solve_ms=[round(v, 3) for v in best[0]],
                                  total=round(sum(best[0]), 3), its=best[1])), flush=True)


if __name__ == "__main__":
    main()
