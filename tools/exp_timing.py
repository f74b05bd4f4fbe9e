"""EXP_finite (fused vs two-pass) and EXP_true at the C4 finest level (512^3) through the C ABI, and the
C4 right-hand side: CUDA-event times, best of 5."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402

if os.environ.get("ECMG_LIB_PATH"):   # A/B timing of a variant build (tuning only)
    ecmg.LIB_PATH = os.environ["ECMG_LIB_PATH"]


def best(fn, reps=5):
    st = torch.cuda.current_stream()
    b = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        b = min(b, e0.elapsed_time(e1))
    return b


def main():
    levels = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    only = sys.argv[2] if len(sys.argv) > 2 else "all"
    g = Grid(4, levels, PROB["C4"])
    L = levels - 1
    w, u2, u4 = g.new_vec(L), g.new_vec(L - 1), g.new_vec(L - 2)
    u2.uniform_(); u4.uniform_()
    ut = g.new_vec(L)
    res = {}
    for fused in (0, 1):
        if only not in ("all", f"exp{fused}"):
            continue
        g.set_option(ecmg.OPT_EXP_KERNEL, fused)
        res[f"exp_finite_fused{fused}_ms"] = best(lambda: g.prolongate_extrapolate(L, u2, u4, w))
    if only in ("all", "run"):   # inside ecmg_run: the free-box output variant, finest level
        u = g.new_vec(L)
        for fused in (0, 1):
            g.set_option(ecmg.OPT_EXP_KERNEL, fused)
            g.run(1e-9, u, ut)
            best_exp = min(g.run(1e-9, u, ut)[1][L]["ms_exp"] for _ in range(3))
            res[f"run_exp_fused{fused}_ms"] = best_exp
            res[f"run_rich_ms"] = g.run(1e-9, u, ut)[1][L]["ms_rich"]
    if only in ("all", "rich"):
        res["exp_true_ms"] = best(lambda: g.richardson(L, w, u2, ut))
    if only in ("all", "rhs"):
        b = g.new_vec(L)
        res["rhs_ms"] = best(lambda: g.level_rhs(L, b))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
