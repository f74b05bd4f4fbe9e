"""C4 (or C3 with --c3) ecmg_run per-level solve time vs ECMG_OPT_PERS_TMA (largest level solved by one cooperative launch of
TMA z-marching passes): CUDA-event TTS, best of 5, plus a tolerance-stopped finest solve from a seeded guess."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402
import synth  # noqa: E402


def main():
    args = sys.argv[1:]
    c3 = "--c3" in args   # C3 (element path, 4^3 -> 256^3, eps 1e-10) instead of C4
    args = [a for a in args if a != "--c3"]
    ths = [int(v) for v in args] or [0, 3000000, 20000000, 200000000]
    L, eps = (7, 1e-10) if c3 else (8, 1e-9)
    g = Grid(4, L, PROB["C3" if c3 else "C4"])
    shape, nodes = g.shape(L - 1)
    u = torch.empty(nodes, dtype=torch.float64, device="cuda")
    ut = torch.empty(nodes, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    x0 = torch.from_numpy(synth.random_nodal(14, shape, (1, 1, 1), tuple(v - 1 for v in shape))).cuda()
    for th in ths + ths:
        g.set_option(ecmg.OPT_PERS_TMA, th)
        g.run(eps, u, ut)
        best, bst = 1e30, None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s, stats = g.run(eps, u, ut)
            e1.record(st)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            if t < best:
                best, bst = t, stats
        x = x0.clone()
        sl = g.solve_level(L - 1, 1e-6, 10000, x)[1]
        ms, it, nf = g.last_jcg_timing()
        print(json.dumps(dict(pers_tma=th, tts=round(best, 3), solve=[round(s["ms_solve"], 3) for s in bst],
                              its=[s["iterations"] for s in bst], fine_solve_ms=round(ms, 3), fine_its=it,
                              ms_per_it=round(ms / max(it, 1), 4))), flush=True)


if __name__ == "__main__":
    main()
