"""ECMG_PROB_ARRAYS (the caller's beta_e, f at the Gauss points, g_D per node and g_R at the
face Gauss points, per level) through the C ABI against the oracle's ARRAYS problem (pinned in
test_oracle_arrays.py), on seeded random data (synth.random_problem_arrays): lifted right-hand side and
operator 1e-13, Alg. 4 iterations +-1 and u, u~ within 1e-9 ||u||_inf (the tolerances of
test_gpu_parity.py). Cases: the element path (random beta, Robin faces with four alphas, a Neumann face),
all-Dirichlet with beta (element path), all-Dirichlet without beta (constant-stencil path); box cells with
free boxes spanning several 32-wide tiles and ragged tails. Also: C3's data sampled into arrays gives the
registry C3's right-hand side on the GPU, and a run is bitwise reproducible."""
import numpy as np
import pytest
import torch

import oracle as o
import synth
from arrays_data import C3_ALPHA, C3_FACES, c3_arrays

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1506_02983_b200 import Grid, PROB, ecmg


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


CASES = {
    "robin": ([1, 1, 1, 1, 0, 0], [2.0, 0.5, 1.5, 3.0, 0.0, 0.0], True),
    "neumann_z": ([0, 0, 0, 1, 0, 1], [0.0, 0.0, 0.0, 0.7, 0.0, 0.0], True),
    "dirichlet_beta": ([0] * 6, [0.0] * 6, True),
    "dirichlet_const": ([0] * 6, [0.0] * 6, False),
    "robin_all": ([1] * 6, [0.5, 1.0, 2.0, 0.25, 1.5, 3.0], True),   # no Dirichlet face at all (still SPD: alpha > 0)
}


def level_data(n0, levels, with_beta, seed=40):
    return [synth.random_problem_arrays(seed + k, tuple(c << k for c in n0), beta=with_beta) for k in range(levels)]


def make(n0, levels, case, data):
    faces, alpha, _ = CASES[case]
    dv = [tuple(dev(a) for a in lv) for lv in data]
    g = Grid(n0, levels, PROB["ARRAYS"], params=alpha, faces=faces, level_arrays=dv)
    return g, dv


@pytest.mark.parametrize("case", list(CASES))
def test_arrays_rhs_and_operator(case):
    n0, levels = (5, 3, 4), 4          # finest 40 x 24 x 32 cells
    faces, alpha, wb = CASES[case]
    data = level_data(n0, levels, wb)
    g, _ = make(n0, levels, case, data)
    for k in (2, 3):
        n = tuple(c << k for c in n0)
        L = o.Level.from_arrays(n, faces, alpha, *data[k])
        free = L.dirichlet()[0] == 0
        b = g.new_vec(k)
        g.level_rhs(k, b)
        bo, _ = L.rhs()
        assert rel(host(b)[free], bo[free]) <= 1e-13
        p = np.where(free, synth.random_nodal(11, n), 0.0)
        q = g.new_vec(k)
        g.apply_operator(k, dev(p), q)
        assert rel(host(q)[free], L.apply(p)[free]) <= 1e-13
    g.close()


@pytest.mark.parametrize("case", list(CASES))
def test_arrays_ecmg_run(case):
    n0, levels, eps = (5, 3, 4), 4, 1e-10
    faces, alpha, wb = CASES[case]
    data = level_data(n0, levels, wb, seed=60)
    g, _ = make(n0, levels, case, data)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(eps, u, ut)
    ost, ostats, ou, out = o.ecmg_arrays(n0, levels, faces, alpha, data, eps)
    assert st == 0 and ost == 0
    it_g = [s["iterations"] for s in stats[2:]]
    it_o = [int(v) for v in ostats[2:, 0]]
    assert all(abs(a - b) <= 1 for a, b in zip(it_g, it_o)), (it_g, it_o)
    assert np.max(np.abs(host(u) - ou)) <= 1e-9 * np.max(np.abs(ou))
    assert np.max(np.abs(host(ut) - out)) <= 1e-9 * np.max(np.abs(out))
    # bitwise reproducible
    u2, ut2 = g.new_vec(levels - 1), g.new_vec(levels - 1)
    g.run(eps, u2, ut2)
    assert torch.equal(u, u2) and torch.equal(ut, ut2)
    g.close()


def test_arrays_sampled_c3_equals_registry():
    n0, levels = (4, 4, 4), 5           # finest 64^3
    data = [c3_arrays((4 << k,) * 3) for k in range(levels)]
    dv = [tuple(dev(a) for a in lv) for lv in data]
    ga = Grid(n0, levels, PROB["ARRAYS"], params=C3_ALPHA, faces=C3_FACES, level_arrays=dv)
    gr = Grid(n0, levels, PROB["C3"])
    k = levels - 1
    ba, br = ga.new_vec(k), gr.new_vec(k)
    ga.level_rhs(k, ba)
    gr.level_rhs(k, br)
    assert rel(host(ba), host(br)) <= 1e-13
    ua, ur = ga.new_vec(k), gr.new_vec(k)
    sa, st_a = ga.run(1e-10, ua)
    sr, st_r = gr.run(1e-10, ur)
    assert sa == 0 and sr == 0
    assert [s["iterations"] for s in st_a] == [s["iterations"] for s in st_r]
    assert rel(host(ua), host(ur)) <= 1e-11
    ga.close()
    gr.close()


def test_arrays_rejects():
    from paper_1506_02983_b200 import ecmg
    data = level_data((4, 4, 4), 3, True)
    dv = [tuple(dev(a) for a in lv) for lv in data]
    with pytest.raises(ecmg.EcmgError):      # alpha < 0
        Grid(4, 3, PROB["ARRAYS"], params=[-1.0, 0, 0, 0, 0, 0], faces=[1, 0, 0, 0, 0, 0], level_arrays=dv)
    with pytest.raises(ecmg.EcmgError):      # beta on some levels only
        dv2 = [dv[0], (None,) + dv[1][1:], dv[2]]
        Grid(4, 3, PROB["ARRAYS"], params=[0.0] * 6, faces=[0] * 6, level_arrays=dv2)
    with pytest.raises(ecmg.EcmgError):      # wrong number of arrays
        Grid(4, 3, PROB["ARRAYS"], params=[0.0] * 6, faces=[0] * 6, level_arrays=dv[:2])


def test_arrays_setup_ahead_bitwise():
    from paper_1506_02983_b200 import ecmg
    n0, levels = (5, 3, 4), 4
    data = level_data(n0, levels, True, seed=80)
    g, _ = make(n0, levels, "robin", data)
    outs = []
    for ahead in (1, 0):
        g.set_option(ecmg.OPT_SETUP_AHEAD, ahead)
        u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
        st, _ = g.run(1e-10, u, ut)
        assert st == 0
        outs.append((u, ut))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    g.close()


def test_arrays_alg3_fixed_schedule():
    # Alg. 3 (Eq. (ee) counts with m_L = 3, ratio 2, plain CG) on ARRAYS data against the oracle
    n0, levels = (5, 3, 4), 4
    faces, alpha, _ = CASES["robin"]
    data = level_data(n0, levels, True, seed=90)
    dv = [tuple(dev(a) for a in lv) for lv in data]
    g = Grid(n0, levels, PROB["ARRAYS"], params=alpha, faces=faces, level_arrays=dv, precond=False)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run_fixed(3, 2.0, u, ut)
    ost, ostats, ou, out = o.ecmg_fixed_arrays(n0, levels, faces, alpha, data, 3, 2.0)
    assert st == 0 and ost == 0
    assert [s["iterations"] for s in stats[2:]] == [int(v) for v in ostats[2:, 0]] == [6, 3]
    assert np.max(np.abs(host(u) - ou)) <= 1e-11 * np.max(np.abs(ou))
    assert np.max(np.abs(host(ut) - out)) <= 1e-11 * np.max(np.abs(out))
    g.close()


def test_arrays_zero_data():
    # no f, g_D, g_R (beta given): b = 0 on every level, so every solve stops before its first iteration
    # (§8c A10) and u = u~ = 0; the oracle agrees
    n0, levels = (4, 4, 4), 4
    faces, alpha = [0, 1, 0, 0, 0, 1], [0.0, 1.5, 0.0, 0.0, 0.0, 0.0]
    data = [(synth.random_problem_arrays(5 + k, (4 << k,) * 3)[0], None, None, None) for k in range(levels)]
    dv = [tuple(dev(a) for a in lv) for lv in data]
    g = Grid(n0, levels, PROB["ARRAYS"], params=alpha, faces=faces, level_arrays=dv)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    u.fill_(1.0)
    ut.fill_(1.0)
    st, stats = g.run(1e-10, u, ut)
    ost, ostats, ou, out = o.ecmg_arrays(n0, levels, faces, alpha, data, 1e-10)
    assert st == 0 and ost == 0
    assert [s["iterations"] for s in stats[2:]] == [int(v) for v in ostats[2:, 0]] == [0, 0]
    assert float(u.abs().max()) == 0.0 and float(ut.abs().max()) == 0.0
    assert np.max(np.abs(ou)) == 0.0
    g.close()


# ---- alpha at the face Gauss points (ARRAYS alpha_q, n_level_arrays = 5 L; Eq. bvp) -------------------
from arrays_data import FACE_AXES, PATCH_FACES, patch_alpha_q, patch_arrays_alpha_q, patch_u, node_points  # noqa: E402


def alpha_q(n, seed):
    """alpha >= 0 at the 4 Gauss points of every face element (gR's layout), seeded."""
    m = sum(4 * n[FACE_AXES[F][0]] * n[FACE_AXES[F][1]] for F in range(6))
    return 3.0 * synth.counter_uniform(seed, m)


@pytest.mark.parametrize("case", ["robin", "neumann_z"])
def test_arrays_alpha_q_rhs_and_operator(case):
    # the Robin mass from alpha_q on the GPU (TMA element kernels, box cells) against the oracle's level
    n0, levels = (5, 3, 4), 4
    faces, alpha, wb = CASES[case]
    data = [lv + (alpha_q(tuple(c << k for c in n0), 90 + k),) for k, lv in enumerate(level_data(n0, levels, wb))]
    g, _ = make(n0, levels, case, data)
    for k in (2, 3):
        n = tuple(c << k for c in n0)
        L = o.Level.from_arrays(n, faces, alpha, *data[k][:4], alpha_q=data[k][4])
        free = L.dirichlet()[0] == 0
        b = g.new_vec(k)
        g.level_rhs(k, b)
        bo, _ = L.rhs()
        assert rel(host(b)[free], bo[free]) <= 1e-13
        p = np.where(free, synth.random_nodal(11, n), 0.0)
        q = g.new_vec(k)
        g.apply_operator(k, dev(p), q)
        assert rel(host(q)[free], L.apply(p)[free]) <= 1e-13
    g.close()


@pytest.mark.parametrize("n0", [(5, 3, 4), (4, 4, 4)])
def test_arrays_alpha_q_ecmg_run(n0):
    # Alg. 4 with alpha_q on every level (one-CTA, cluster / cooperative and TMA solves on the way) vs the oracle
    levels, eps, case = 4, 1e-10, "robin"
    faces, alpha, wb = CASES[case]
    data = [lv + (alpha_q(tuple(c << k for c in n0), 70 + k),) for k, lv in enumerate(level_data(n0, levels, wb, seed=60))]
    g, _ = make(n0, levels, case, data)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(eps, u, ut)
    ost, ostats, ou, out = o.ecmg_arrays(n0, levels, faces, alpha, data, eps)
    assert st == 0 and ost == 0
    it_g = [s["iterations"] for s in stats[2:]]
    it_o = [int(v) for v in ostats[2:, 0]]
    assert all(abs(a - b) <= 1 for a, b in zip(it_g, it_o)), (it_g, it_o)
    assert np.max(np.abs(host(u) - ou)) <= 1e-9 * np.max(np.abs(ou))
    assert np.max(np.abs(host(ut) - out)) <= 1e-9 * np.max(np.abs(out))
    g.close()


def test_arrays_alpha_q_patch_exact():
    # the layered linear patch with random alpha_q >= 0 on four Robin faces: the FE solution is u itself (Galerkin
    # exactness, pinned for the oracle in test_oracle_arrays.py), on every path of the cascade to 64^3
    n0, levels = 4, 5
    lv = []
    for k in range(levels):
        n = (n0 << k,) * 3
        lv.append(patch_arrays_alpha_q(n, np.full(n[2], 1.3), patch_alpha_q(n)))
    dv = [tuple(dev(a) for a in x) for x in lv]
    g = Grid(n0, levels, PROB["ARRAYS"], params=[0.0] * 6, faces=PATCH_FACES, level_arrays=dv)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(1e-13, u, ut)
    assert st == 0
    nf = (n0 << (levels - 1),) * 3
    ue = patch_u(*node_points(nf, (0, 0, 0), (1, 1, 1))).reshape(-1)
    assert np.max(np.abs(host(u) - ue)) <= 1e-10 and np.max(np.abs(host(ut) - ue)) <= 1e-10
    g.close()


def test_arrays_shifted_box_domain():
    # a domain that is not the unit cube (shifted and stretched box, anisotropic cells): C3's data sampled on it,
    # Alg. 4 on the GPU against the oracle on the same box (grid coordinates lo + i h with h = (hi - lo) / n)
    lo, hi = (-0.5, 0.0, 0.25), (1.5, 0.75, 1.0)
    n0, levels, eps = (4, 3, 2), 4, 1e-10
    data = [c3_arrays(tuple(c << k for c in n0), lo, hi) for k in range(levels)]
    dv = [tuple(dev(a) for a in lv) for lv in data]
    g = Grid(n0, levels, PROB["ARRAYS"], params=C3_ALPHA, faces=C3_FACES, level_arrays=dv, lo=lo, hi=hi)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(eps, u, ut)
    ost, ostats, ou, out = o.ecmg_arrays(n0, levels, C3_FACES, C3_ALPHA, data, eps, lo=lo, hi=hi)
    assert st == 0 and ost == 0
    it_g = [s["iterations"] for s in stats[2:]]
    it_o = [int(v) for v in ostats[2:, 0]]
    assert all(abs(a - b) <= 1 for a, b in zip(it_g, it_o)), (it_g, it_o)
    assert np.max(np.abs(host(u) - ou)) <= 1e-9 * np.max(np.abs(ou))
    assert np.max(np.abs(host(ut) - out)) <= 1e-9 * np.max(np.abs(out))
    g.close()


@pytest.mark.parametrize("pid", ["C1", "PATCH_TRILINEAR"])
def test_registry_problem_on_shifted_box(pid):
    # the registry problems on a shifted box: the GPU evaluates f, g_D at lo + i h exactly as the oracle does
    lo, hi = (0.25, -1.0, 0.5), (1.25, 0.5, 2.5)
    n0, levels, eps = (4, 4, 4), 4, 1e-9
    p = PROB[pid]
    g = Grid(n0, levels, p, lo=lo, hi=hi)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(eps, u, ut)
    ost, ostats, ou, out = o.ecmg(n0, levels, p, eps, lo=lo, hi=hi)
    assert st == 0 and ost == 0
    it_g = [s["iterations"] for s in stats[2:]]
    it_o = [int(v) for v in ostats[2:, 0]]
    assert all(abs(a - b) <= 1 for a, b in zip(it_g, it_o)), (it_g, it_o)
    assert np.max(np.abs(host(u) - ou)) <= 1e-9 * np.max(np.abs(ou))
    assert np.max(np.abs(host(ut) - out)) <= 1e-9 * np.max(np.abs(out))
    g.close()


@pytest.mark.parametrize("case,P", [("robin", 2), ("neumann_z", 4), ("dirichlet_const", 8)])
def test_arrays_on_virtual_slabs(case, P):
    # the caller's data on z-slabs: every slab reads its planes of the global-domain arrays (alpha_q included),
    # P slabs against the oracle; levels with 32 or more z cells split
    n0, levels, eps = (4, 4, 4), 5, 1e-10
    faces, alpha, wb = CASES[case]
    data = [lv + (alpha_q(tuple(c << k for c in n0), 110 + k),) for k, lv in enumerate(level_data(n0, levels, wb, seed=80))]
    g, _ = make(n0, levels, case, data)
    g.set_option(ecmg.OPT_VIRTUAL_SLABS, P)
    g.set_option(ecmg.OPT_SHARD_MIN, 16)
    u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
    st, stats = g.run(eps, u, ut)
    ost, ostats, ou, out = o.ecmg_arrays(n0, levels, faces, alpha, data, eps)
    assert st == 0 and ost == 0
    it_g = [s["iterations"] for s in stats[2:]]
    it_o = [int(v) for v in ostats[2:, 0]]
    assert all(abs(a - b) <= 1 for a, b in zip(it_g, it_o)), (it_g, it_o)
    assert np.max(np.abs(host(u) - ou)) <= 1e-9 * np.max(np.abs(ou))
    assert np.max(np.abs(host(ut) - out)) <= 1e-9 * np.max(np.abs(out))
    g.close()
