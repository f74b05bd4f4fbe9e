"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: C4 (configs[3],
4^3 -> 512^3, the default bench line; constant-stencil TMA kernels), C3 (configs[2], 256^3; element-beta
kernels with a Robin face) and C5 (configs[4], 1024^3, layered geology: right-hand side, EXP_finite, operator,
one JCG iteration, EXP_true). The assembled oracle does not fit in host memory at these sizes, so outputs are
sampled (random nodes plus the domain faces and the 32-wide tile seams of the kernels) and the oracle
computes them one row / node at a time (oracle.rows, oracle.exp_nodes: pinned bitwise to the assembled
oracle in test_oracle_rows.py). Where an output depends on global sums (a CG step, a whole solve), the
test checks properties that hold at any size: the step is alpha * p0 with p0 = D^-1 (b - A x0) from the
oracle's rows and one alpha for every node; the solve meets its stopping test, is deterministic, and its
errors against the exact solution fall at the expected orders from 256^3 to 512^3.
Inputs: synth's seeded vectors (seeds 11 p, 12 u_4h, 13 u_2h, 14 x0; §8d T1)."""
import numpy as np
import pytest
import torch

import oracle as o
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1506_02983_b200 import Grid, ecmg


def sample_nodes(n, count, seed):
    """Random nodes plus nodes on / next to the domain faces and on both sides of the kernels' 32-wide
    tile seams (free-box x / y index 31 | 32, i.e. node 32 | 33)."""
    rng = np.random.default_rng(seed)
    pts = [rng.integers(0, np.array(n) + 1, size=(count, 3))]
    edge = np.array([0, 1, 2, n[0] - 2, n[0] - 1, n[0]])
    k = count // 4
    for d in range(3):
        p = rng.integers(0, np.array(n) + 1, size=(k, 3))
        p[:, d] = rng.choice(edge, size=k)
        pts.append(p)
    seam = np.array([31, 32, 33, 34, 63, 64, 65, 66])
    p = rng.integers(0, np.array(n) + 1, size=(k, 3))
    p[:, 0] = rng.choice(seam, size=k)
    p[:, 1] = rng.choice(seam, size=k)
    pts.append(p)
    return np.unique(np.concatenate(pts), axis=0)


def lin(n, nodes):
    return nodes[:, 0] + (n[0] + 1) * (nodes[:, 1] + (n[1] + 1) * nodes[:, 2])


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host_at(t, idx):
    torch.cuda.synchronize()
    return t[torch.from_numpy(idx).cuda()].cpu().numpy()


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


CFG = {"c4": (o.C4, 8, (512,) * 3), "c3": (o.C3, 7, (256,) * 3)}


@pytest.fixture(scope="module", params=["c4", "c3"])
def level(request):
    pid, levels, n = CFG[request.param]
    g = Grid(4, levels, pid)
    nodes = sample_nodes(n, 3000, 7)
    yield pid, levels, n, g, nodes
    g.close()
    torch.cuda.empty_cache()


def test_fullsize_rhs(level):
    pid, levels, n, g, nodes = level
    b = g.new_vec(levels - 1)
    g.level_rhs(levels - 1, b)
    _, bo = o.rows(n, pid, nodes)
    assert rel(host_at(b, lin(n, nodes)), bo) <= 1e-13


def test_fullsize_rhs_c4_symmetric_load():
    # the permutation-symmetric C4 load (k_rhs_c4_sym, the bench's default at 512^3 and 256^3): (a) every node of
    # the level against the plain kernel (ECMG_OPT_RHS_SYM = 0) -- a tile that is not written, written twice or
    # written with the wrong image shows up here; (b) nodes on both sides of its 31-node tile seams along every
    # axis, in every class of tile triple, against the oracle's rows
    pid, levels, n = o.C4, 8, (512,) * 3
    for lv in (levels - 1, levels - 2):
        g = Grid(4, lv + 1, pid)
        b1 = g.new_vec(lv)
        g.level_rhs(lv, b1)
        g.set_option(ecmg.OPT_RHS_SYM, 0)
        b0 = g.new_vec(lv)
        g.level_rhs(lv, b0)
        torch.cuda.synchronize()
        d = float((b1 - b0).abs().max() / b0.abs().max())
        print(f"C4 load at {4 << lv}^3: symmetric vs plain kernel, max rel diff {d:.2e}")
        assert d <= 1e-14
        assert not torch.equal(b1, b0)   # (the two kernels do differ in rounding order: both really ran)
        if lv == levels - 1:
            rng = np.random.default_rng(31)
            seams = np.concatenate([31 * np.arange(1, 17), 31 * np.arange(1, 17) + 1])   # free index 31k-1 | 31k
            pts = rng.choice(seams, size=(4000, 3))
            pts[:1000, 2] = rng.integers(1, 512, size=1000)      # seams in x, y only
            pts[1000:2000, 0] = rng.integers(1, 512, size=1000)  # seams in y, z only
            nodes = np.unique(pts, axis=0)
            _, bo = o.rows(n, pid, nodes)
            assert rel(host_at(b1, lin(n, nodes)), bo) <= 1e-13
        g.close()
        del b0, b1
        torch.cuda.empty_cache()


def test_fullsize_stencil_apply(level):
    pid, levels, n, g, nodes = level
    p = synth.random_nodal(11, n)
    q = g.new_vec(levels - 1)
    g.apply_operator(levels - 1, dev(p), q)
    qo, _ = o.rows(n, pid, nodes, p)
    assert rel(host_at(q, lin(n, nodes)), qo) <= 1e-13


def test_fullsize_one_jcg_iteration(level):
    # x1 - x0 = alpha p0 with p0 = D^-1 (b - A x0): the TMA K1 / K2 kernels of the bench's fixed-iteration
    # run, checked node by node against the oracle's rows; alpha is a global ratio, so every sampled node
    # must give the same one
    pid, levels, n, g, nodes = level
    x0 = synth.random_nodal(14, n)
    x = dev(x0)
    st, s = g.solve_level(levels - 1, 0.0, 1, x)
    assert st == 0 and s["iterations"] == 1
    idx = lin(n, nodes)
    ax, b, dg = o.rows(n, pid, nodes, x0, diag=True)
    free = dg > 0
    p0 = (b[free] - ax[free]) / dg[free]
    dx = host_at(x, idx)[free] - x0[idx][free]
    big = np.abs(p0) >= 1e-2 * np.max(np.abs(p0))
    alpha = dx[big] / p0[big]
    assert alpha.size > 100
    a0 = np.median(alpha)
    assert np.max(np.abs(alpha - a0)) <= 1e-10 * abs(a0), (alpha.min(), alpha.max())
    assert rel(dx, a0 * p0) <= 1e-10


def test_fullsize_exp_finite(level):
    pid, levels, n, g, nodes = level
    n2, n4 = tuple(c // 2 for c in n), tuple(c // 4 for c in n)
    u2, u4 = synth.random_nodal(13, n2), synth.random_nodal(12, n4)
    w = g.new_vec(levels - 1)
    g.prolongate_extrapolate(levels - 1, dev(u2), dev(u4), w)
    wo = o.exp_nodes(n, pid, 0, u2, u4, nodes)
    assert rel(host_at(w, lin(n, nodes)), wo) <= 1e-14


def test_fullsize_exp_true(level):
    pid, levels, n, g, nodes = level
    uh, u2 = synth.random_nodal(11, n), synth.random_nodal(13, tuple(c // 2 for c in n))
    ut = g.new_vec(levels - 1)
    g.richardson(levels - 1, dev(uh), dev(u2), ut)
    uto = o.exp_nodes(n, pid, 2, uh, u2, nodes)
    assert rel(host_at(ut, lin(n, nodes)), uto) <= 1e-14


def exact_on_device(pid, n):
    """u on every node of the level (the problem's exact solution, evaluated on the device)."""
    z, y, x = torch.meshgrid(*[torch.arange(c + 1, dtype=torch.float64, device="cuda") / c for c in n[::-1]],
                             indexing="ij")
    if pid == o.C4:
        return (x * x + y * y + z * z) ** 0.75
    return torch.cos(np.pi * x) * torch.cos(np.pi * y) * torch.exp(z)


def test_fullsize_ecmg_run_bench_config():
    # the bench's step (ecmg_run, C4 4^3 -> 512^3, eps = 1e-9, default options): every level meets its
    # stopping test and the run is bitwise reproducible
    pid, levels, n = CFG["c4"]
    g = Grid(4, levels, pid)
    runs = []
    for _ in range(2):
        u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
        st, stats = g.run(1e-9, u, ut)
        assert st == 0
        assert all(s["converged"] for s in stats)
        assert all(s["rel_res_recur"] <= 1e-9 for s in stats[2:])
        assert stats[-1]["rel_res_true"] <= 1e-8
        runs.append(([s["iterations"] for s in stats], u, ut))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1]) and torch.equal(runs[0][2], runs[1][2])
    # the default run forms u~_h inside the finest level's true-residual pass (ECMG_OPT_RICH_FUSED); the separate
    # EXP_true kernel gives the same u~_h bit for bit, and u_h / the counts are untouched
    g.set_option(ecmg.OPT_RICH_FUSED, 0)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(1e-9, u, ut)
    assert st == 0 and [s["iterations"] for s in stats] == runs[0][0]
    assert torch.equal(u, runs[0][1]) and torch.equal(ut, runs[0][2])
    g.close()
    del runs, u, ut
    torch.cuda.empty_cache()


def test_fullsize_orders():
    # the same cascade with a tight tolerance (eps = 1e-12, so the algebraic error is below the
    # discretisation error; at the bench's 1e-9 it is not): from 256^3 to 512^3 the RMS error of
    # u_h falls at order 2 and that of u~_h at order ~3, the order the paper reports for solutions of this
    # regularity (u = r^{3/2} in H^{3-eps}; Table 10). Measured: 1.99 and 2.87.
    pid = o.C4
    rms = []
    for lv in (7, 8):
        g = Grid(4, lv, pid)
        u, ut = g.new_vec(lv - 1), g.new_vec(lv - 1)
        st, stats = g.run(1e-12, u, ut)
        assert st == 0
        ue = exact_on_device(pid, (4 << (lv - 1),) * 3).reshape(-1)
        rms.append((float((u - ue).pow(2).mean().sqrt()), float((ut - ue).pow(2).mean().sqrt())))
        del u, ut, ue
        g.close()
        torch.cuda.empty_cache()
    (eu2, et2), (eu1, et1) = rms
    assert 1.8 <= np.log2(eu2 / eu1) <= 2.2, rms
    assert np.log2(et2 / et1) >= 2.6, rms
    assert et1 < 0.05 * eu1, rms


def test_fullsize_c5():
    # C5 (configs[4], layered geology, 4^3 -> 1024^3, element beta): the finest right-hand side, EXP_finite,
    # the operator, one JCG iteration and EXP_true on sampled nodes against the oracle's one-row / one-node evaluations
    pid, levels = o.C5, 9
    n = (1024,) * 3
    prm = synth.c5_geometry(0)
    g = Grid(4, levels, pid, prm)
    nodes = sample_nodes(n, 2000, 9)
    idx = lin(n, nodes)
    b = g.new_vec(levels - 1)
    g.level_rhs(levels - 1, b)
    _, bo = o.rows(n, pid, nodes, params=prm)
    assert rel(host_at(b, idx), bo) <= 1e-13
    del b
    n2, n4 = tuple(c // 2 for c in n), tuple(c // 4 for c in n)
    u2, u4 = synth.random_nodal(13, n2), synth.random_nodal(12, n4)
    w = g.new_vec(levels - 1)
    g.prolongate_extrapolate(levels - 1, dev(u2), dev(u4), w)
    wo = o.exp_nodes(n, pid, 0, u2, u4, nodes, params=prm)
    assert rel(host_at(w, idx), wo) <= 1e-14
    del w, u2, u4
    g.close()
    torch.cuda.empty_cache()


def test_fullsize_c5_operator_and_iteration():
    # the element operator, one JCG iteration and EXP_true at 1024^3 (the bench's jcg_fixed_c5 kernels) need
    # the seeded 8.6 GB input and its generator's temporaries on the host
    import psutil
    avail = psutil.virtual_memory().available
    if avail < 96 << 30:
        pytest.skip(f"host has {avail / 2**30:.0f} GiB available, the 1024^3 seeded input needs ~96 GiB")
    pid, levels = o.C5, 9
    n = (1024,) * 3
    prm = synth.c5_geometry(0)
    g = Grid(4, levels, pid, prm)
    nodes = sample_nodes(n, 2000, 9)
    idx = lin(n, nodes)
    n2 = tuple(c // 2 for c in n)
    p = synth.random_nodal(11, n)
    q = g.new_vec(levels - 1)
    g.apply_operator(levels - 1, dev(p), q)
    qo, _ = o.rows(n, pid, nodes, p, params=prm)
    assert rel(host_at(q, idx), qo) <= 1e-13
    del q
    x = dev(p)
    st, s = g.solve_level(levels - 1, 0.0, 1, x)
    assert st == 0 and s["iterations"] == 1
    ax, bb, dg = o.rows(n, pid, nodes, p, params=prm, diag=True)
    free = dg > 0
    p0 = (bb[free] - ax[free]) / dg[free]
    dx = host_at(x, idx)[free] - p[idx][free]
    big = np.abs(p0) >= 1e-2 * np.max(np.abs(p0))
    alpha = dx[big] / p0[big]
    a0 = np.median(alpha)
    assert alpha.size > 100 and np.max(np.abs(alpha - a0)) <= 1e-10 * abs(a0)
    del x
    u2 = synth.random_nodal(13, n2)
    ut = g.new_vec(levels - 1)
    g.richardson(levels - 1, dev(p), dev(u2), ut)
    uto = o.exp_nodes(n, pid, 2, p, u2, nodes, params=prm)
    assert rel(host_at(ut, idx), uto) <= 1e-14
    del ut, u2, p
    g.close()
    torch.cuda.empty_cache()
