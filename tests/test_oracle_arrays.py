"""The oracle's ARRAYS problem (SURVEY.md §8b ECMG_PROB_ARRAYS: beta_e, f at the Gauss points, g_D per node,
g_R at the face Gauss points, given by the caller per level) pinned against what fixes it independently:
(1) C3's data sampled at those points gives the level the analytic C3 registry builds (matrix, load, lifted
right-hand side, Dirichlet values), which test_oracle_fe.py pins to closed forms; a transposed array
index (element order, Gauss point order, face block or in-face order) moves values by O(h) and fails it;
(2) a layered-beta linear patch with Robin faces of four different alphas is solved exactly (Galerkin
exactness: u is in the Q1 space and beta grad u is divergence free), which fails for a wrong beta layer or a
misplaced g_R block; (3) Alg. 4 on the sampled C3 reproduces Alg. 4 on the analytic C3."""
import numpy as np
import pytest

import oracle as o
import synth
from arrays_data import C3_ALPHA, C3_FACES, PATCH_ALPHA, PATCH_FACES, c3_arrays, patch_arrays, patch_u, node_points


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("n,lo,hi", [((6, 5, 4), (0, 0, 0), (1, 1, 1)), ((4, 6, 8), (-0.5, 0.0, 0.25), (1.5, 0.75, 1.0))])
def test_sampled_c3_equals_registry(n, lo, hi):
    ref = o.Level(n, o.C3, lo=lo, hi=hi)
    arr = o.Level.from_arrays(n, C3_FACES, C3_ALPHA, *c3_arrays(n, lo, hi), lo=lo, hi=hi)
    assert rel(arr.matrix(), ref.matrix()) <= 1e-14
    assert rel(arr.load(), ref.load()) <= 1e-13
    (ba, na), (br, nr) = arr.rhs(), ref.rhs()
    assert rel(ba, br) <= 1e-13 and abs(na - nr) <= 1e-13 * nr
    (ma, ga), (mr, gr) = arr.dirichlet(), ref.dirichlet()
    assert np.array_equal(ma, mr) and rel(ga, gr) <= 1e-15


def test_arrays_none_defaults():
    # beta = 1, f = g_D = g_R = 0 when the arrays are absent: the Laplacian with a zero right-hand side
    n = (4, 3, 5)
    a = o.Level.from_arrays(n, [0, 1, 0, 0, 1, 0], [0, 0.5, 0, 0, 2.0, 0])
    assert np.max(np.abs(a.rhs()[0])) == 0.0 and np.max(np.abs(a.load())) == 0.0
    one = o.Level.from_arrays(n, [0, 1, 0, 0, 1, 0], [0, 0.5, 0, 0, 2.0, 0], beta_e=np.ones(60))
    assert np.array_equal(a.matrix(), one.matrix())


def test_arrays_reject():
    with pytest.raises(ValueError):
        o.Level.from_arrays((4, 4, 4), [0] * 6, [0, 0, -1.0, 0, 0, 0])   # alpha < 0


@pytest.mark.parametrize("n", [(4, 4, 4), (6, 5, 7)])
def test_layered_patch_exact(n):
    layer = 0.5 + 1.5 * synth.counter_uniform(31, n[2])
    L = o.Level.from_arrays(n, PATCH_FACES, PATCH_ALPHA, *patch_arrays(n, layer))
    x, s = L.jcg(np.zeros(L.N), 1e-14, 10000)
    assert s["status"] == 0
    free = L.dirichlet()[0] == 0
    ue = patch_u(*node_points(n, (0, 0, 0), (1, 1, 1))).reshape(-1)
    assert np.max(np.abs(x - ue)[free]) <= 1e-11


def test_layered_patch_wrong_layer_order_fails():
    # the same data with the element layers reversed is a different problem: the patch is no longer exact
    n = (4, 4, 6)
    layer = 0.5 + 1.5 * synth.counter_uniform(31, n[2])
    b, f, g, r = patch_arrays(n, layer)
    L = o.Level.from_arrays(n, PATCH_FACES, PATCH_ALPHA, b.reshape(n[2], -1)[::-1].reshape(-1), f, g, r)
    x, _ = L.jcg(np.zeros(L.N), 1e-14, 10000)
    free = L.dirichlet()[0] == 0
    ue = patch_u(*node_points(n, (0, 0, 0), (1, 1, 1))).reshape(-1)
    assert np.max(np.abs(x - ue)[free]) > 1e-6


def test_ecmg_arrays_equals_registry():
    lv = 4
    arrays = [c3_arrays((4 << k,) * 3) for k in range(lv)]
    sa, ta, ua, uta = o.ecmg_arrays(4, lv, C3_FACES, C3_ALPHA, arrays, 1e-10)
    sr, tr, ur, utr = o.ecmg(4, lv, o.C3, 1e-10)
    assert sa == 0 and sr == 0
    assert list(ta[:, 0]) == list(tr[:, 0])
    assert rel(ua, ur) <= 1e-11 and rel(uta, utr) <= 1e-11


def test_ecmg_fixed_arrays_equals_registry():
    # Alg. 3 (fixed counts, plain CG) on the sampled C3 = Alg. 3 on the registry C3
    lv = 4
    arrays = [c3_arrays((4 << k,) * 3) for k in range(lv)]
    sa, ta, ua, uta = o.ecmg_fixed_arrays(4, lv, C3_FACES, C3_ALPHA, arrays, 3, 2.0)
    sr, tr, ur, utr = o.ecmg_fixed(4, lv, o.C3, 3, 2.0)
    assert sa == 0 and sr == 0
    assert list(ta[:, 0]) == list(tr[:, 0])
    assert rel(ua, ur) <= 1e-11 and rel(uta, utr) <= 1e-11


# ---- alpha at the face Gauss points (ARRAYS alpha_q; Eq. bvp) -------------------------------------------
from arrays_data import FACE_AXES, patch_alpha_q, patch_arrays_alpha_q  # noqa: E402


def test_alpha_q_constant_equals_per_face_alpha():
    # alpha_q = alpha_F at every Gauss point of face F is the per-face-alpha level, bit for bit (matrix, load, b)
    n = (5, 4, 6)
    layer = 0.5 + 1.5 * synth.counter_uniform(31, n[2])
    arrs = patch_arrays(n, layer)
    aq = np.concatenate([np.full(4 * n[FACE_AXES[F][0]] * n[FACE_AXES[F][1]], PATCH_ALPHA[F]) for F in range(6)])
    a = o.Level.from_arrays(n, PATCH_FACES, PATCH_ALPHA, *arrs)
    q = o.Level.from_arrays(n, PATCH_FACES, [0.0] * 6, *arrs, alpha_q=aq)
    assert np.array_equal(a.matrix(), q.matrix()) and np.array_equal(a.load(), q.load())
    assert np.array_equal(a.rhs()[0], q.rhs()[0])


@pytest.mark.parametrize("n", [(4, 4, 4), (6, 5, 7)])
def test_alpha_q_patch_exact(n):
    # random alpha_q >= 0 on four Robin faces, g_R consistent at the same Gauss points: u stays the exact FE solution
    layer = 0.5 + 1.5 * synth.counter_uniform(31, n[2])
    aq = patch_alpha_q(n)
    L = o.Level.from_arrays(n, PATCH_FACES, [0.0] * 6, *patch_arrays_alpha_q(n, layer, aq)[:4], alpha_q=aq)
    x, s = L.jcg(np.zeros(L.N), 1e-14, 10000)
    assert s["status"] == 0
    free = L.dirichlet()[0] == 0
    ue = patch_u(*node_points(n, (0, 0, 0), (1, 1, 1))).reshape(-1)
    assert np.max(np.abs(x - ue)[free]) <= 1e-11


def test_alpha_q_is_used():
    # the alpha_q patch data with the per-face alphas instead of alpha_q is a different problem: not exact
    n = (5, 5, 4)
    layer = 0.5 + 1.5 * synth.counter_uniform(31, n[2])
    aq = patch_alpha_q(n)
    b, f, g, r, _ = patch_arrays_alpha_q(n, layer, aq)
    L = o.Level.from_arrays(n, PATCH_FACES, PATCH_ALPHA, b, f, g, r)
    x, _ = L.jcg(np.zeros(L.N), 1e-14, 10000)
    free = L.dirichlet()[0] == 0
    ue = patch_u(*node_points(n, (0, 0, 0), (1, 1, 1))).reshape(-1)
    assert np.max(np.abs(x - ue)[free]) > 1e-6


def test_alpha_q_symmetric_spd():
    n = (4, 5, 3)
    aq = patch_alpha_q(n)
    L = o.Level.from_arrays(n, PATCH_FACES, [0.0] * 6, alpha_q=aq)
    A = L.matrix()
    # the band matrix is symmetric: entry (i, slot) equals entry (j, mirrored slot)
    nn = (n[0] + 1, n[1] + 1, n[2] + 1)
    free = L.dirichlet()[0] == 0
    dense = np.zeros((L.N, L.N))
    for i in range(L.N):
        ix, iy, iz = i % nn[0], (i // nn[0]) % nn[1], i // (nn[0] * nn[1])
        for s in range(27):
            dx, dy, dz = s % 3 - 1, (s // 3) % 3 - 1, s // 9 - 1
            jx, jy, jz = ix + dx, iy + dy, iz + dz
            if 0 <= jx < nn[0] and 0 <= jy < nn[1] and 0 <= jz < nn[2]:
                dense[i, jx + nn[0] * (jy + nn[1] * jz)] = A[i, s]
    Af = dense[np.ix_(free, free)]
    assert np.array_equal(Af, Af.T)
    assert np.all(np.linalg.eigvalsh(Af) > 0)


def test_ecmg_arrays_alpha_q_patch():
    # Alg. 4 on the alpha_q patch (alpha_q on every level): u_h and u~_h equal the linear u on the finest level
    n0, levels = 4, 4
    lv = []
    for k in range(levels):
        n = (n0 << k,) * 3
        layer = 0.5 + 1.5 * synth.counter_uniform(31, n[2])
        lv.append(patch_arrays_alpha_q(n, np.repeat(layer[:1], n[2]), patch_alpha_q(n)))
    st, stats, u, ut = o.ecmg_arrays(n0, levels, PATCH_FACES, [0.0] * 6, lv, 1e-13)
    assert st == 0
    nf = (n0 << (levels - 1),) * 3
    ue = patch_u(*node_points(nf, (0, 0, 0), (1, 1, 1))).reshape(-1)
    assert np.max(np.abs(u - ue)) <= 1e-10 and np.max(np.abs(ut - ue)) <= 1e-10
