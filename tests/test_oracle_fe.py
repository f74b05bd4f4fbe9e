"""Pins for the oracle's FE discretisation (§2) -- closed forms, invariants, Galerkin
exactness. Kinds per SURVEY.md §8c C.3. No GPU."""
import numpy as np
import pytest

import oracle as o
import synth


def slot(dx, dy, dz):
    return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)


# --- element stiffness (Eq. for a(u,v)) ----------------------------------------------

def test_element_stiffness_cube_closed_form():
    # closed form on a cube of side h: K = beta*(h/12)*{4 same, 0 one axis differs, -1 two/three differ}
    for h in (1.0, 0.25, 1.0 / 512):
        K = o.element_stiffness([h, h, h], 1.0)
        for a in range(8):
            for b in range(8):
                nd = bin(a ^ b).count("1")
                expect = {0: 4.0, 1: 0.0, 2: -1.0, 3: -1.0}[nd] * h / 12.0
                assert abs(K[a, b] - expect) <= 1e-15 * h
    K1 = o.element_stiffness([1, 1, 1], 1.0)
    assert np.allclose(np.diag(K1), 1.0 / 3.0, rtol=0, atol=1e-15)
    assert np.allclose(K1.sum(axis=1), 0.0, atol=1e-15)                # S:119 row sums 0
    assert np.array_equal(K1, K1.T)
    K2 = o.element_stiffness([2, 2, 2], 1.0)
    assert np.allclose(K2, 2 * K1, rtol=1e-15, atol=1e-15)             # S:123 scaling
    assert np.all(o.element_stiffness([1, 1, 1], 0.0) == 0.0)          # beta = 0


def test_element_stiffness_box_analytic():
    # analytic integral for a box: K = V * sum_d (1/h_d^2) k_d (x) m (x) m with 1D
    # k = [[1,-1],[-1,1]], m = [[1/3,1/6],[1/6,1/3]] (exact integrals of trilinear shape functions)
    h = np.array([0.1, 0.25, 0.2])
    V = h.prod()
    k = np.array([[1.0, -1.0], [-1.0, 1.0]])
    m = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    K = o.element_stiffness(h, 2.5)
    for a in range(8):
        for b in range(8):
            ad = [(a >> d) & 1 for d in range(3)]
            bd = [(b >> d) & 1 for d in range(3)]
            val = 0.0
            for d in range(3):
                t = k[ad[d], bd[d]] / h[d] ** 2
                for e in range(3):
                    if e != d:
                        t *= m[ad[e], bd[e]]
                val += t
            assert abs(K[a, b] - 2.5 * V * val) < 1e-14


def test_face_integrals_closed_form():
    one = np.ones(4)
    M, G = o.face_integrals(1.0, 1.0, one, np.zeros(4))   # diagonal 1/9
    for c in range(4):
        for d in range(4):
            nd = bin(c ^ d).count("1")
            assert abs(M[c, d] - {0: 1 / 9, 1: 1 / 18, 2: 1 / 36}[nd]) < 1e-16
    M0, G1 = o.face_integrals(1.0, 1.0, np.zeros(4), one)  # load 1/4 each
    assert np.all(M0 == 0.0)
    assert np.allclose(G1, 0.25, atol=1e-16)


# --- assembled operator -------------------------------------------------------------------------

def test_global_stencil_beta1_cube():
    # interior row: 8h/3 centre, 0 faces, -h/6 edges, -h/12 corners
    n = 8
    h = 1.0 / n
    L = o.Level((n, n, n), o.C1)
    A = L.matrix().reshape(n + 1, n + 1, n + 1, 27)
    row = A[4, 4, 4]
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                k = abs(dx) + abs(dy) + abs(dz)
                expect = {0: 8 * h / 3, 1: 0.0, 2: -h / 6, 3: -h / 12}[k]
                assert abs(row[slot(dx, dy, dz)] - expect) < 1e-15
    assert abs(row.sum()) < 1e-15


@pytest.mark.parametrize("pid,n", [(o.C3, (8, 8, 8)), (o.C5, (8, 8, 8)), (o.P1, (8, 8, 8)), (o.P2, (10, 4, 5))])
def test_assembled_symmetric_bitwise(pid, n):
    params = synth.c5_geometry(0) if pid == o.C5 else None
    L = o.Level(n, pid, params=params)
    A = L.matrix()
    nx, ny, nz = (v + 1 for v in n)
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                i = ix + nx * (iy + ny * iz)
                for dz in (-1, 0, 1):
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            jx, jy, jz = ix + dx, iy + dy, iz + dz
                            if not (0 <= jx < nx and 0 <= jy < ny and 0 <= jz < nz):
                                assert A[i, slot(dx, dy, dz)] == 0.0
                                continue
                            j = jx + nx * (jy + ny * jz)
                            assert A[i, slot(dx, dy, dz)] == A[j, slot(-dx, -dy, -dz)]  # bitwise


def test_load_f1_is_h3():
    # f = 1: each element entry is V/8, an interior node collects 8 of them -> h^3
    n = 8
    L = o.Level((n, n, n), o.CONST_F)
    F = L.load().reshape(n + 1, n + 1, n + 1)
    assert np.allclose(F[1:-1, 1:-1, 1:-1], 1.0 / n ** 3, rtol=1e-14, atol=0)
    assert abs(F[0, 0, 0] - 1.0 / n ** 3 / 8) < 1e-18


def test_robin_plane_stencil():
    # Robin face z=1 with alpha=1, beta=1: row of a free Robin node = half of the volume stencil
    # plus the assembled face-mass stencil 4h^2/9 (centre), h^2/9 (axis), h^2/36 (diagonal)
    n = 8
    h = 1.0 / n
    L = o.Level((n, n, n), o.PATCH_ROBIN)
    A = L.matrix().reshape(n + 1, n + 1, n + 1, 27)
    row = A[n, 4, 4]
    Kc = o.element_stiffness([h, h, h])
    # volume part: 4 elements below the face contribute (local a at az=1)
    vol = np.zeros(27)
    for ex in (-1, 0):
        for ey in (-1, 0):
            a = (0 if ex == 0 else 1) + 2 * (0 if ey == 0 else 1) + 4
            for b in range(8):
                dx = (b & 1) - (a & 1)
                dy = ((b >> 1) & 1) - ((a >> 1) & 1)
                dz = ((b >> 2) & 1) - ((a >> 2) & 1)
                vol[slot(dx, dy, dz)] += Kc[a, b]
    face = np.zeros(27)
    face[slot(0, 0, 0)] = 4 * h * h / 9
    for d in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        face[slot(d[0], d[1], 0)] = h * h / 9
    for d in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
        face[slot(d[0], d[1], 0)] = h * h / 36
    assert np.allclose(row, vol + face, rtol=0, atol=1e-15)


def test_spd_small():
    # Cholesky of A_ff succeeds (dsolve raises otherwise) on 4^3 / 8^3 / 16^3
    for n in (4, 8, 16):
        o.Level((n, n, n), o.C3).dsolve()
    o.Level((8, 8, 8), o.C5, params=synth.c5_geometry(0)).dsolve()


# --- Galerkin exactness (patch tests) -------------------------------------------

@pytest.mark.parametrize("pid,params", [
    (o.PATCH_TRILINEAR, None),
    (o.PATCH_LAYERED, synth.layered_only(0)),
    (o.PATCH_ROBIN, None),
    (o.PATCH_ROBIN_XY, None),   # Robin on the four side faces, four different alphas, edges shared by two
])
def test_patch_exact(pid, params):
    L = o.Level((8, 8, 8), pid, params=params)
    ue = L.exact()
    u = L.dsolve()
    assert np.max(np.abs(u - ue)) <= 1e-12 * max(1.0, np.max(np.abs(ue)))
    x, st = L.jcg(np.zeros(L.N), 1e-14, 10000)
    assert st["status"] == 0
    assert np.max(np.abs(x - ue)) <= 1e-12 * max(1.0, np.max(np.abs(ue)))


def test_free_node_count_p1():
    # P1 on 8^3: 729 - 217 = 512 free nodes
    m, _ = o.Level((8, 8, 8), o.P1).dirichlet()
    assert int((~m).sum()) == 512


def test_c5_fixture_matches_generator():
    import json, os
    d = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c5_seed0.json")))
    p = synth.c5_geometry(0)
    flat = d["heights"] + d["layer_beta"] + sum(d["boxes"], []) + d["x0"] + [d["sigma"], d["amplitude"]]
    assert np.array_equal(np.array(flat), p)
    assert np.all(np.diff(d["heights"]) > 0)
    assert all(0.1 <= b <= 10 for b in d["layer_beta"])
