"""Pins for the oracle's JCG / CG (Alg. 4 l.7-9) and DSOLVE:
brute-force direct solves, textbook reductions and invariants (SURVEY.md §8c C.3 'O7')."""
import numpy as np
import pytest

import oracle as o
import synth


@pytest.mark.parametrize("pid,n", [(o.C2, 4), (o.C2, 8), (o.C3, 8), (o.C5, 8), (o.P1, 8), (o.P2, (10, 4, 5))])
def test_jcg_matches_cholesky(pid, n):
    n3 = (n, n, n) if np.isscalar(n) else n
    params = synth.c5_geometry(0) if pid == o.C5 else None
    L = o.Level(n3, pid, params=params)
    xd = L.dsolve()
    x, st = L.jcg(np.zeros(L.N), 1e-14, 10000)
    assert st["status"] == 0
    assert np.max(np.abs(x - xd)) <= 1e-10 * np.max(np.abs(xd))
    # the direct solve satisfies the system to rounding
    b, nb = L.rhs()
    m, g = L.dirichlet()
    r = (b - L.apply(np.where(m, 0.0, xd)))[~m]
    assert np.linalg.norm(r) <= 1e-13 * nb


def test_dense_numpy_cross_check():
    # independent dense solve with numpy on the same assembled A_ff (brute force, 4^3)
    L = o.Level((4, 4, 4), o.C3)
    m, g = L.dirichlet()
    free = np.flatnonzero(~m)
    E = np.zeros((L.N, free.size))
    E[free, np.arange(free.size)] = 1.0
    Aff = np.stack([L.apply(E[:, k]) for k in range(free.size)], axis=1)[free]
    b, _ = L.rhs()
    xs = np.linalg.solve(Aff, b[free])
    xd = L.dsolve()[free]
    assert np.max(np.abs(xs - xd)) <= 1e-12 * np.max(np.abs(xs))
    assert np.allclose(Aff, Aff.T, rtol=0, atol=0)
    assert np.all(np.linalg.eigvalsh(Aff) > 0)


def test_zero_rhs_zero_iterations():
    p = synth.c5_geometry(0)
    p[47] = 0.0  # zero source amplitude, homogeneous Dirichlet: b = 0
    L = o.Level((8, 8, 8), o.C5, params=p)
    x, st = L.jcg(np.zeros(L.N), 1e-10, 100)
    assert st["iterations"] == 0 and st["status"] == 0 and np.all(x == 0)


def test_converged_guess_zero_iterations():
    L = o.Level((8, 8, 8), o.C1)
    xd = L.dsolve()
    x, st = L.jcg(xd, 1e-8, 100)
    assert st["iterations"] == 0   # §8c A10: loop test before the first iteration


def test_energy_norm_monotone():
    # A-norm of the error is non-increasing along CG/JCG
    L = o.Level((8, 8, 8), o.C5, params=synth.c5_geometry(0))
    m, _ = L.dirichlet()
    xs = L.dsolve()
    prev = np.inf
    first = None
    for k in range(0, 40):
        x, _ = L.jcg(np.zeros(L.N), 0.0, k)
        e = np.where(m, 0.0, x - xs)
        en = float(e @ L.apply(e))
        first = en if first is None else first
        assert en <= prev * (1 + 1e-12) + 1e-24 * first   # until rounding level
        prev = en


def test_jcg_equals_cg_constant_diagonal():
    # beta = 1, cubic cells, pure Dirichlet: diag(A_ff) = (8h/3) I, so JCG == CG iterate by iterate
    # in exact arithmetic
    L = o.Level((16, 16, 16), o.C2)
    x0 = synth.random_nodal(14, (16, 16, 16), (1, 1, 1), (15, 15, 15))
    for k in (1, 5, 20):
        xj, _ = L.jcg(x0, 0.0, k, precond=True)
        xc, _ = L.jcg(x0, 0.0, k, precond=False)
        assert np.max(np.abs(xj - xc)) <= 1e-12 * np.max(np.abs(xc))


def test_jacobi_helps_with_neumann():
    # P1 has Neumann faces, so diag(A_ff) is not constant and JCG differs from CG; the paper
    # reports JCG <= CG iterations per level (Tables 1-3).
    L = o.Level((16, 16, 16), o.P1)
    _, sj = L.jcg(np.zeros(L.N), 1e-8, 1000, precond=True)
    _, sc = L.jcg(np.zeros(L.N), 1e-8, 1000, precond=False)
    assert sj["iterations"] < sc["iterations"]


def test_rel_true_reported():
    L = o.Level((8, 8, 8), o.C3)
    x, st = L.jcg(np.zeros(L.N), 1e-9, 1000)
    b, nb = L.rhs()
    m, _ = L.dirichlet()
    r = (b - L.apply(np.where(m, 0.0, x)))[~m]
    assert abs(np.linalg.norm(r) / nb - st["rel_true"]) <= 1e-13
    assert st["rel_recur"] <= 1e-9
    assert np.all(x[m] == L.dirichlet()[1][m])  # Dirichlet entries = g_D


def test_alg3_fixed_schedule():
    # Alg. 3 / Eq. (ee): m_j = ceil(m_L ratio^(L-j)); the paper's suggested m_j = 4 * 4^(L-j)
    st, S, u, ut = o.ecmg_fixed(4, 5, o.C2, 4, 4.0)
    assert st == 0
    assert [int(v) for v in S[2:, 0]] == [64, 16, 4]
    # zero iterations: u_h is W_h = EXP_finite(u_2h, u_4h) exactly
    st, S, u0, ut0, w0 = o.ecmg_fixed(4, 4, o.C2, 0, 2.0, want_w=True)
    assert np.array_equal(u0, w0) and int(S[-1, 0]) == 0
    # enough iterations: Alg. 3 reaches the same FE solution as Alg. 4 at a tight tolerance
    st, S, ua, _ = o.ecmg_fixed(4, 4, o.C2, 200, 1.0, precond=True)
    st2, S2, ub, _ = o.ecmg(4, 4, o.C2, 1e-13)
    assert np.max(np.abs(ua - ub)) <= 1e-11 * np.max(np.abs(ub))
