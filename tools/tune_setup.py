"""C4 / C3 ecmg_run time-to-solution vs the setup-ahead knobs (ECMG_OPT_SETUP_AHEAD, ECMG_OPT_SETUP_CTAS),
CUDA events on the grid's stream, best of 5 after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402


def tts(g, eps, u, ut, reps=5):
    st = torch.cuda.current_stream()
    best, stats = 1e30, None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s, stats = g.run(eps, u, ut)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, stats


def main():
    ctas = [int(v) for v in sys.argv[1:]] or [0, 1, 2, 3]
    for name, pid, levels, eps in (("c4", PROB["C4"], 8, 1e-9), ("c3", PROB["C3"], 7, 1e-10)):
        g = Grid(4, levels, pid)
        shape, nodes = g.shape(levels - 1)
        u = torch.empty(nodes, dtype=torch.float64, device="cuda")
        ut = torch.empty(nodes, dtype=torch.float64, device="cuda")
        for ahead, c in [(0, 0), (1, 0), (0, 0), (1, 0), (1, 0)]:
            g.set_option(ecmg.OPT_SETUP_AHEAD, ahead)
            g.set_option(ecmg.OPT_SETUP_CTAS, c)
            g.run(eps, u, ut)
            t, stats = tts(g, eps, u, ut)
            print(json.dumps(dict(cfg=name, ahead=ahead, ctas=c, tts=round(t, 3),
                                  solve=[round(s["ms_solve"], 3) for s in stats],
                                  wait=[round(s["ms_setup"], 3) for s in stats])), flush=True)
        g.close()


if __name__ == "__main__":
    main()
