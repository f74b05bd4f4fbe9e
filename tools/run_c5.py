"""One full-size C5 run (BASELINE configs[4]: layered geology, seed 0, 4^3 -> 1024^3, eps 1e-8, element-beta
path): per-level iterations and times, TTS. Not a bench line (the driver's bench is C4)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1506_02983_b200 import Grid, PROB  # noqa: E402


def main():
    levels = int(sys.argv[1]) if len(sys.argv) > 1 else 9
    fly = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    g = Grid(4, levels, PROB["C5"], synth.c5_geometry(0))
    from paper_1506_02983_b200 import ecmg
    g.set_option(ecmg.OPT_BETA_FLY, fly)
    shape, nodes = g.shape(levels - 1)
    u = torch.empty(nodes, dtype=torch.float64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t0 = time.time()
    ev[0].record()
    st, stats = g.run(1e-8, u)
    ev[1].record()
    torch.cuda.synchronize()
    out = dict(config="C5 4^3->%d^3" % (4 << (levels - 1)), beta_fly=fly, status=st, tts_ms=ev[0].elapsed_time(ev[1]),
               wall_s=time.time() - t0, iterations=[s["iterations"] for s in stats],
               solve_ms=[round(s["ms_solve"], 2) for s in stats], rel_true=[s["rel_res_true"] for s in stats],
               mem_gb=torch.cuda.max_memory_allocated() / 1e9)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
