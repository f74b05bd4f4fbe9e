"""Pins for the oracle's EXP_finite (Eqs. jiedian, zhongdian, sifen1/2, inter) and
EXP_true (Eqs. t1, chenlin): the printed worked example, a hand-derived
symmetry-class table, polynomial exactness, and exact h^2-expansion identities."""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as o
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
LABELS = o.SEED_LABELS


def nat(label):
    t = label - 1
    return ((t % 5) - 2) / 2.0, (((t // 5) % 5) - 2) / 2.0, ((t // 25) - 2) / 2.0


def test_w35_worked_example():
    w = o.serendipity_weights(*nat(35))
    assert nat(35) == (1.0, -0.5, -0.5)
    g = GOLD["w35"]
    expect = {lab: float(Fraction(v)) for lab, v in zip(g["labels"], g["weights"])}
    for s, lab in enumerate(LABELS):
        assert w[s] == expect.get(lab, 0.0), lab   # bitwise


# Hand-derived representative rows of the 8 symmetry classes of the 105 non-seed nodes
# (derived from N_i of P:494-501, independent of the code). Keys are natural
# coordinates of seeds; unlisted seeds have weight 0.
F = Fraction
CLASSES = {
    (F(-1, 2), -1, -1): {(-1, -1, -1): F(3, 8), (0, -1, -1): F(3, 4), (1, -1, -1): F(-1, 8)},
    (1, 0, 0): {(1, 0, 1): F(1, 2), (1, 0, -1): F(1, 2), (1, 1, 0): F(1, 2), (1, -1, 0): F(1, 2),
                (1, 1, 1): F(-1, 4), (1, 1, -1): F(-1, 4), (1, -1, 1): F(-1, 4), (1, -1, -1): F(-1, 4)},
    (1, F(1, 2), 0): {(1, 1, 1): F(-3, 16), (1, 1, -1): F(-3, 16), (1, -1, 1): F(-3, 16), (1, -1, -1): F(-3, 16),
                      (1, 0, 1): F(3, 8), (1, 0, -1): F(3, 8), (1, 1, 0): F(3, 4), (1, -1, 0): F(1, 4)},
    (1, F(-1, 2), F(-1, 2)): {(1, 0, -1): F(9, 16), (1, -1, 0): F(9, 16), (1, 0, 1): F(3, 16), (1, 1, 0): F(3, 16),
                              (1, 1, -1): F(-3, 16), (1, -1, 1): F(-3, 16), (1, 1, 1): F(-1, 8)},
    (0, 0, 0): "body",
    (F(1, 2), 0, 0): "axis",
    (F(1, 2), F(1, 2), 0): "facediag",
    (F(1, 2), F(1, 2), F(1, 2)): "diag",
}


def _seed_coords():
    return [tuple(F(int(2 * c), 2) for c in nat(l)) for l in LABELS]


def _rep_weights(rep, spec):
    seeds = _seed_coords()
    if isinstance(spec, dict):
        return {tuple(F(c) for c in k): v for k, v in spec.items()}
    w = {}
    for s in seeds:
        nmid = sum(1 for c in s if c == 0)
        if spec == "body":
            w[s] = F(1, 4) if nmid == 1 else F(-1, 4)
        elif spec == "axis":  # (1/2,0,0)
            if nmid == 0:
                w[s] = F(-9, 32) if s[0] == 1 else F(-5, 32)
            elif s[0] == 0:
                w[s] = F(3, 16)
            else:
                w[s] = F(3, 8) if s[0] == 1 else F(1, 8)
        elif spec == "facediag":  # (1/2,1/2,0)
            if nmid == 0:
                pos = (s[0] == 1) + (s[1] == 1)
                w[s] = {2: F(-9, 32), 1: F(-3, 16), 0: F(-3, 32)}[pos]
            elif s[0] == 0:
                w[s] = F(9, 32) if s[1] == 1 else F(3, 32)
            elif s[1] == 0:
                w[s] = F(9, 32) if s[0] == 1 else F(3, 32)
            else:
                pos = (s[0] == 1) + (s[1] == 1)
                w[s] = {2: F(9, 16), 1: F(3, 16), 0: F(1, 16)}[pos]
        elif spec == "diag":  # (1/2,1/2,1/2)
            if nmid == 0:
                pos = sum(1 for c in s if c == 1)
                w[s] = {3: F(-27, 128), 2: F(-27, 128), 1: F(-15, 128), 0: F(-7, 128)}[pos]
            else:
                f = F(3, 16)
                for c in s:
                    if c != 0:
                        f *= (1 + F(c, 2))
                w[s] = f
    return w


def test_serendipity_class_table_bitwise():
    seeds = _seed_coords()
    seen = {}
    for rep, spec in CLASSES.items():
        rep = tuple(F(c) for c in rep)
        wrep = _rep_weights(rep, spec)
        assert sum(wrep.values()) == 1
        for perm in itertools.permutations(range(3)):
            for sg in itertools.product((1, -1), repeat=3):
                tr = lambda p: tuple(sg[i] * p[perm[i]] for i in range(3))
                node = tr(rep)
                wn = {tr(k): v for k, v in wrep.items()}
                if node in seen:
                    assert seen[node] == wn
                seen[node] = wn
    assert len(seen) == 105   # 24+6+24+24+1+6+12+8
    for node, wn in seen.items():
        w = o.serendipity_weights(*(float(c) for c in node))
        for s, sc in enumerate(seeds):
            assert w[s] == float(wn.get(sc, 0)), (node, sc)   # bitwise
    # seed rows are unit rows
    for s, lab in enumerate(LABELS):
        w = o.serendipity_weights(*nat(lab))
        assert np.array_equal(w, np.eye(20)[s])


def _grid_fn(n, fn):
    x = np.arange(n + 1) / n
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    return fn(X, Y, Z).reshape(-1)


def _free(L):
    m, _ = L.dirichlet()
    return ~m


QUAD = lambda X, Y, Z: 0.3 + X - 2 * Y + 0.5 * Z + X * X - 3 * Y * Y + 2 * Z * Z + X * Y - Y * Z + 4 * X * Z \
    + X * Y * Z + X * X * Y - Y * Y * Z + Z * Z * X + 2 * X * X * Y * Z   # in the 20-dim Serendipity space


@pytest.mark.parametrize("variant", [0, 1])
def test_exp_finite_reproduces_serendipity_space(variant):
    # U^0 = U^1 = nodal samples of q: seeds reduce to q and W = q at every node
    n = 16
    L = o.Level((n, n, n), o.C1)
    q = QUAD if variant == 0 else (lambda X, Y, Z: QUAD(X, Y, Z) + X * X * Y * Y * Z * Z)  # Lagrange: 27-dim
    u2, u4, uf = _grid_fn(n // 2, q), _grid_fn(n // 4, q), _grid_fn(n, q)
    w = L.exp_finite(u2, u4, variant)
    fr = _free(L)
    assert np.max(np.abs(w[fr] - uf[fr])) <= 1e-13


@pytest.mark.parametrize("variant", [0, 1])
def test_exp_finite_h2_expansion_exact(variant):
    # U^i = q + c 4^(2-i) (an exact h^2 expansion): W = q + c at every free node (derived)
    n, c = 16, 0.37
    L = o.Level((n, n, n), o.C1)
    u2 = _grid_fn(n // 2, QUAD) + 4 * c
    u4 = _grid_fn(n // 4, QUAD) + 16 * c
    w = L.exp_finite(u2, u4, variant)
    fr = _free(L)
    assert np.max(np.abs(w[fr] - (_grid_fn(n, QUAD) + c)[fr])) <= 1e-13


def test_exp_finite_constants():
    n = 16
    L = o.Level((n, n, n), o.C1)
    w = L.exp_finite(np.ones((n // 2 + 1) ** 3), np.zeros((n // 4 + 1) ** 3))
    fr = _free(L)
    assert np.allclose(w[fr], 1.25, rtol=0, atol=1e-15)
    m, g = L.dirichlet()
    assert np.array_equal(w[m], g[m])                    # Dirichlet overwrite (§8c A15)


def test_exp_finite_quarter_points_sifen():
    # on coarse edges the trace is 1D quadratic interpolation: Eqs. (sifen1)/(sifen2)
    n = 16
    L = o.Level((n, n, n), o.PATCH_ROBIN, faces=[1] * 6)   # all Robin: no Dirichlet overwrite
    u2 = synth.random_nodal(13, (n // 2,) * 3)
    u4 = synth.random_nodal(12, (n // 4,) * 3)
    w = L.exp_finite(u2, u4).reshape(n + 1, n + 1, n + 1)
    U1 = u2.reshape((n // 2 + 1,) * 3)
    U0 = u4.reshape((n // 4 + 1,) * 3)
    for bz, by, bx in [(0, 0, 0), (1, 2, 3), (3, 3, 3)]:
        # x-edge at (y, z) = (4by, 4bz): nodes x = 4bx..4bx+4
        j, jm, j1 = 2 * bx, 2 * bx + 1, 2 * bx + 2
        a1, m1, b1 = U1[2 * bz, 2 * by, j], U1[2 * bz, 2 * by, jm], U1[2 * bz, 2 * by, j1]
        a0, b0 = U0[bz, by, bx], U0[bz, by, bx + 1]
        s1 = ((9 * a1 + 12 * m1 - b1) - (3 * a0 + b0)) / 16
        s2 = ((9 * b1 + 12 * m1 - a1) - (3 * b0 + a0)) / 16
        assert abs(w[4 * bz, 4 * by, 4 * bx + 1] - s1) < 1e-14
        assert abs(w[4 * bz, 4 * by, 4 * bx + 3] - s2) < 1e-14


def test_exp_finite_linear():
    n = 16
    L = o.Level((n, n, n), o.C1)
    a2, a4 = synth.random_nodal(13, (8,) * 3), synth.random_nodal(12, (4,) * 3)
    b2, b4 = synth.random_nodal(23, (8,) * 3), synth.random_nodal(22, (4,) * 3)
    m, _ = L.dirichlet()
    wa, wb = L.exp_finite(a2, a4), L.exp_finite(b2, b4)
    wab = L.exp_finite(2 * a2 - 3 * b2, 2 * a4 - 3 * b4)
    assert np.max(np.abs((wab - (2 * wa - 3 * wb))[~m])) < 1e-13


# --- EXP_true --------------------------------------------------------------------------------

def test_exp_true_constant():
    n = 8
    L = o.Level((n, n, n), o.PATCH_ROBIN, faces=[1] * 6)
    ut = L.exp_true(np.full(L.N, 3.0), np.zeros((n // 2 + 1) ** 3))
    assert np.allclose(ut, 4.0, rtol=0, atol=1e-15)


def test_exp_true_exact_expansion_any_q():
    # U^1 = q + c, U^0 = q + 4c for ANY nodal q: u~ = q exactly (derived from Eqs. t1, chenlin)
    n, c = 16, -0.61
    L = o.Level((n, n, n), o.PATCH_ROBIN, faces=[1] * 6)
    q = synth.random_nodal(11, (n,) * 3)
    q2 = q.reshape((n + 1,) * 3)[::2, ::2, ::2].reshape(-1)
    ut = L.exp_true(q + c, q2 + 4 * c)
    assert np.max(np.abs(ut - q)) < 1e-14


def test_exp_true_same_samples_identity():
    n = 8
    L = o.Level((n, n, n), o.PATCH_ROBIN, faces=[1] * 6)
    f = _grid_fn(n, QUAD)
    ut = L.exp_true(f, _grid_fn(n // 2, QUAD))
    assert np.max(np.abs(ut - f)) < 1e-14


def test_exp_true_trilinear_closed_form():
    # derived identity: u~ = u_h + (1/3) I_trilinear(u_h|_2h - u_2h),
    # evaluated here by an independent numpy trilinear interpolation
    n = 8
    L = o.Level((n, n, n), o.PATCH_ROBIN, faces=[1] * 6)
    uh = synth.random_nodal(11, (n,) * 3)
    u2 = synth.random_nodal(13, (n // 2,) * 3)
    d = uh.reshape((n + 1,) * 3)[::2, ::2, ::2] - u2.reshape((n // 2 + 1,) * 3)
    I = np.zeros((n + 1,) * 3)
    for k in range(n + 1):
        for j in range(n + 1):
            for i in range(n + 1):
                k0, j0, i0 = min(k // 2, n // 2 - 1), min(j // 2, n // 2 - 1), min(i // 2, n // 2 - 1)
                tz, ty, tx = (k - 2 * k0) / 2, (j - 2 * j0) / 2, (i - 2 * i0) / 2
                v = 0.0
                for a, wz in ((0, 1 - tz), (1, tz)):
                    for b, wy in ((0, 1 - ty), (1, ty)):
                        for cc, wx in ((0, 1 - tx), (1, tx)):
                            v += wz * wy * wx * d[k0 + a, j0 + b, i0 + cc]
                I[k, j, i] = v
    ut = L.exp_true(uh, u2)
    assert np.max(np.abs(ut - (uh + I.reshape(-1) / 3))) < 1e-14
