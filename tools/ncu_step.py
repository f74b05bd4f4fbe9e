"""Profiling driver for ncu: one warm-up ECMG_jcg run on C4 (512^3), then -- between
cudaProfilerStart/Stop -- one full ECMG run and `--iters` fixed fine-grid JCG iterations.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/ncu_step.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1506_02983_b200 import Grid, PROB  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--skip-run", action="store_true")
    ap.add_argument("--host-loop", action="store_true",
                    help="JCG loop driven from the host (same kernels): ncu does not list launches inside the "
                         "CUDA graph's conditional WHILE body")
    ap.add_argument("--unfused", action="store_true",
                    help="the fixed iterations run the unfused textbook PCG sequence (ECMG_OPT_UNFUSED ablation)")
    a = ap.parse_args()
    pid, n0, levels, eps = {"c4": (PROB["C4"], 4, 8, 1e-9), "c3": (PROB["C3"], 4, 7, 1e-10),
                            "c2": (PROB["C2"], 4, 6, 1e-10)}[a.config]
    g = Grid(n0, levels, pid)
    if a.host_loop:
        from paper_1506_02983_b200 import ecmg
        g.set_option(ecmg.OPT_GRAPH, 0)
    shape, nodes = g.shape(levels - 1)
    u = torch.empty(nodes, dtype=torch.float64, device="cuda")
    ut = torch.empty_like(u)
    g.run(eps, u, ut)
    x0 = torch.from_numpy(synth.random_nodal(14, shape, (1, 1, 1), tuple(v - 1 for v in shape))).cuda()
    if a.unfused:
        from paper_1506_02983_b200 import ecmg as _e
        g.set_option(_e.OPT_UNFUSED, 1)
    g.solve_level(levels - 1, 0.0, 2, x0.clone())
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    if not a.skip_run:
        st, stats = g.run(eps, u, ut)
    g.solve_level(levels - 1, 0.0, a.iters, x0.clone())
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ncu_step done", [s["iterations"] for s in stats] if not a.skip_run else "")


if __name__ == "__main__":
    main()
