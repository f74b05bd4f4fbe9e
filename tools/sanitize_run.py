"""Small runs of every kernel family for compute-sanitizer: memcheck / racecheck / synccheck
over 16^3 - 64^3 levels. Paths: the one-CTA solve, the cooperative register-resident solve, the cooperative TMA
solve, the TMA K1/K2 graph loop and host loop (constant and element operators), EXP_finite (fused and two-pass,
both variants), EXP_true, the setup kernels, the virtual-slab path with fused peer halo stores, and ARRAYS data.
Usage: python tools/sanitize_run.py [small] [--guards]   (small: 16^3 / 32^3 only; --guards: run against
libecmg_test.so and check the guard bands around every library buffer and around the caller's vectors)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1506_02983_b200 import Grid, PROB, ecmg  # noqa: E402

small = "small" in sys.argv[1:]
guards = "--guards" in sys.argv[1:]
if guards:   # the -DECMG_TESTING build: guard bands around every device buffer of the library
    ecmg.LIB_PATH = os.path.join(os.path.dirname(ecmg.LIB_PATH), "libecmg_test.so")
torch.cuda.set_device(0)
GB = 4096          # guard doubles around the caller's output vectors
SENTINEL = -7.25e301
bad_total = 0


def guarded_vec(g, level):
    """A caller vector inside a larger tensor whose head and tail hold a sentinel (out-of-bounds writes into
    the caller's buffer change them)."""
    _, nodes = g.shape(level)
    buf = torch.full((nodes + 2 * GB,), SENTINEL, dtype=torch.float64, device="cuda")
    return buf, buf[GB:GB + nodes]


def check(name, bufs):
    global bad_total
    torch.cuda.synchronize()
    bad = 0
    for b in bufs:
        bad += int((b[:GB] != SENTINEL).sum()) + int((b[-GB:] != SENTINEL).sum())
    if guards:
        fn = ecmg.lib().ecmg_test_guard_check
        fn.restype = ctypes.c_longlong
        bad += int(fn())
    bad_total += bad
    print(f"   {name}: corrupted guard entries {bad}", flush=True)


def run(name, pid, levels, eps, opts=(), params=None, variant=0, fixed=None):
    g = Grid(4, levels, pid, params, exp_variant=variant)
    for o, v in opts:
        g.set_option(o, v)
    bu, u = guarded_vec(g, levels - 1)
    but, ut = guarded_vec(g, levels - 1)
    if fixed:
        st, stats = g.run_fixed(fixed[0], fixed[1], u, ut)
    else:
        st, stats = g.run(eps, u, ut)
    torch.cuda.synchronize()
    print(f"{name}: status {st} iterations {[s['iterations'] for s in stats]}", flush=True)
    # a race shows up as run-to-run differences: 5 more runs must repeat u_h and u~_h bit for bit
    u0, ut0 = u.clone(), ut.clone()
    global bad_total
    for _ in range(5):
        if fixed:
            g.run_fixed(fixed[0], fixed[1], u, ut)
        else:
            g.run(eps, u, ut)
        torch.cuda.synchronize()
        nd = int((u != u0).sum()) + int((ut != ut0).sum())
        if nd:
            print(f"   {name}: NOT bitwise reproducible ({nd} entries differ)", flush=True)
            bad_total += nd
    # the single-level entry points on the finest level: solve, apply, EXP_finite, EXP_true, rhs
    k = levels - 1
    bw, w = guarded_vec(g, k)
    b2, u2 = guarded_vec(g, k - 1)
    b4, u4 = guarded_vec(g, k - 2)
    u2.uniform_()
    u4.uniform_()
    g.prolongate_extrapolate(k, u2, u4, w)
    g.richardson(k, u, u2, ut)
    g.apply_operator(k, u, w)
    g.level_rhs(k, w)
    g.solve_level(k, 0.0, 3, u)
    check(name, [bu, but, bw, b2, b4])
    g.close()
    check(name + " (after destroy)", [])


c5 = synth.c5_geometry(0)
L = 4 if small else 5   # finest 32^3 or 64^3
# default ladder: one-CTA (<= 8^3), register-resident cooperative (16^3, 32^3), cooperative TMA (64^3)
run("C4 default", PROB["C4"], L, 1e-9)
run("C3 default (element path, Robin)", PROB["C3"], L, 1e-10)
run("C5 default (element path)", PROB["C5"], L, 1e-8, params=c5)
run("C1 Lagrange EXP", PROB["C1"], L, 1e-8, variant=1)
# TMA K1/K2 kernels: CUDA-graph WHILE loop and host loop (persistent paths off)
off = [(ecmg.OPT_PERSISTENT, 0), (ecmg.OPT_PERS_TMA, 0), (ecmg.OPT_CTA_SOLVE, 0)]
run("C2 graph loop (TMA K1/K2)", PROB["C2"], L, 1e-10, off)
run("C3 graph loop (element TMA K1/K2)", PROB["C3"], L, 1e-10, off)
run("C2 host loop", PROB["C2"], L, 1e-10, off + [(ecmg.OPT_GRAPH, 0)])
run("C4 register-prefetch kernels", PROB["C4"], L, 1e-9, off + [(ecmg.OPT_KERNEL, 0)])
run("C4 two-pass EXP", PROB["C4"], L, 1e-9, [(ecmg.OPT_EXP_KERNEL, 0)])
run("C4 setup in line", PROB["C4"], L, 1e-9, [(ecmg.OPT_SETUP_AHEAD, 0)])
run("C2 Alg. 3 fixed counts, plain CG", PROB["C2"], L, 0.0, [(ecmg.OPT_PRECOND, 0)], fixed=(3, 2.0))
# z-slabs on one GPU (device copies for the halo messages), copied and fused peer halo stores
for fused in (0, 1):
    run(f"C4 virtual slabs P=2 fused_halo={fused}", PROB["C4"], L, 1e-9,
        [(ecmg.OPT_VIRTUAL_SLABS, 2), (ecmg.OPT_SHARD_MIN, 16), (ecmg.OPT_FUSED_HALO, fused)])
    run(f"C5 virtual slabs P=4 fused_halo={fused}", PROB["C5"], L, 1e-8,
        [(ecmg.OPT_VIRTUAL_SLABS, 4), (ecmg.OPT_SHARD_MIN, 16), (ecmg.OPT_FUSED_HALO, fused)], params=c5)
# ARRAYS: the caller's data (C4 sampled at the points the discretisation reads)
import bench  # noqa: E402
n0, lv = 4, L
arrs = bench.c4_level_arrays(n0, lv)
dev = [(fq.cuda(), gd.cuda()) for fq, gd in arrs]
ga = Grid(n0, lv, PROB["ARRAYS"], params=[0.0] * 6, faces=[0] * 6, level_arrays=[(None, f, g, None) for f, g in dev])
u, ut = ga.new_vec(lv - 1), ga.new_vec(lv - 1)
st, stats = ga.run(1e-9, u, ut)
torch.cuda.synchronize()
print(f"C4 as ARRAYS: status {st} iterations {[s['iterations'] for s in stats]}", flush=True)
ga.close()
check("C4 as ARRAYS", [])
print(f"sanitize_run done: corrupted guard entries or irreproducible entries {bad_total}", flush=True)
sys.exit(1 if bad_total else 0)
