"""Data of the ARRAYS problem (SURVEY.md §8b ECMG_PROB_ARRAYS) sampled from analytic problems at the points
the discretisation reads: beta at element centroids (reading A3), f at the 2x2x2 Gauss points of
each element, g_D at the nodes, g_R at the 2x2 Gauss points of each face element. Test input builders: the
sampled C3 (Eq. (bvp) data of BASELINE.json's C3, written out here in numpy) and a layered-beta linear patch
with Robin faces whose Q1 solution is exact."""
import numpy as np

G = 0.57735026918962576451   # 1/sqrt(3)
FACE_AXES = [(1, 2), (1, 2), (0, 2), (0, 2), (0, 1), (0, 1)]   # in-face axes d1 < d2 of faces x-, x+, y-, y+, z-, z+


def _grid_1d(lo, h, n, offs):
    """lo + (e + off) h for e = 0..n-1 and each offset (last axis)."""
    return lo + (np.arange(n)[:, None] + np.asarray(offs)[None, :]) * h


def element_points(n, lo, hi):
    """(cx, cy, cz) centroids [nz, ny, nx] and Gauss points (x, y, z) [nz, ny, nx, 8] with q = qx + 2qy + 4qz."""
    h = [(hi[d] - lo[d]) / n[d] for d in range(3)]
    offs = [(1.0 - G) / 2.0, (1.0 + G) / 2.0]
    c = [lo[d] + (np.arange(n[d]) + 0.5) * h[d] for d in range(3)]
    gp = [_grid_1d(lo[d], h[d], n[d], offs) for d in range(3)]   # [n_d, 2]
    q = np.arange(8)
    X = gp[0][None, None, :, q & 1]
    Y = gp[1][None, :, None, (q >> 1) & 1]
    Z = gp[2][:, None, None, (q >> 2) & 1]
    X, Y, Z = np.broadcast_arrays(X, Y, Z)
    cz, cy, cx = np.meshgrid(c[2], c[1], c[0], indexing="ij")
    return (cx, cy, cz), (X, Y, Z)


def node_points(n, lo, hi):
    z, y, x = np.meshgrid(*[lo[d] + np.arange(n[d] + 1) * (hi[d] - lo[d]) / n[d] for d in (2, 1, 0)], indexing="ij")
    return x, y, z


def face_points(n, lo, hi, F):
    """Gauss points of face F's elements: coordinate arrays [n_d2, n_d1, 4], q = q1 + 2 q2."""
    d = F // 2
    d1, d2 = FACE_AXES[F]
    h = [(hi[k] - lo[k]) / n[k] for k in range(3)]
    offs = [(1.0 - G) / 2.0, (1.0 + G) / 2.0]
    g1 = _grid_1d(lo[d1], h[d1], n[d1], offs)
    g2 = _grid_1d(lo[d2], h[d2], n[d2], offs)
    q = np.arange(4)
    P = [None] * 3
    P[d1] = np.broadcast_to(g1[None, :, q & 1], (n[d2], n[d1], 4))
    P[d2] = np.broadcast_to(g2[:, None, (q >> 1) & 1], (n[d2], n[d1], 4))
    P[d] = np.full((n[d2], n[d1], 4), hi[d] if F & 1 else lo[d])
    return P


def sample(n, lo, hi, beta, f, gD, gR, faces):
    """ARRAYS data of one level: beta(x,y,z) at centroids, f at Gauss points, gD at nodes, gR(F, x, y, z) at the
    face Gauss points of the Robin faces (0 on the other faces' blocks)."""
    (cx, cy, cz), (X, Y, Z) = element_points(n, lo, hi)
    b = beta(cx, cy, cz).reshape(-1) if beta is not None else None
    fq = f(X, Y, Z).reshape(-1)
    g = gD(*node_points(n, lo, hi)).reshape(-1)
    blocks = []
    for F in range(6):
        P = face_points(n, lo, hi, F)
        blocks.append((gR(F, *P) if faces[F] == 1 else np.zeros_like(P[0])).reshape(-1))
    return b, fq, g, np.concatenate(blocks)


# ---- C3 (BASELINE.json configs[2]): u = cos(pi x) cos(pi y) e^z, beta = 1 + 0.5 sin(2 pi x) cos(2 pi y) sin(2 pi z),
#      Robin z = 1 with alpha = 1: g_R = alpha u + beta du/dz = (1 + beta) u
def c3_u(x, y, z):
    return np.cos(np.pi * x) * np.cos(np.pi * y) * np.exp(z)


def c3_beta(x, y, z):
    return 1.0 + 0.5 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y) * np.sin(2 * np.pi * z)


def c3_f(x, y, z):
    u, b = c3_u(x, y, z), c3_beta(x, y, z)
    bx = np.pi * np.cos(2 * np.pi * x) * np.cos(2 * np.pi * y) * np.sin(2 * np.pi * z)
    by = -np.pi * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    bz = np.pi * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y) * np.cos(2 * np.pi * z)
    ux = -np.pi * np.sin(np.pi * x) * np.cos(np.pi * y) * np.exp(z)
    uy = -np.pi * np.cos(np.pi * x) * np.sin(np.pi * y) * np.exp(z)
    return -b * (1.0 - 2.0 * np.pi ** 2) * u - (bx * ux + by * uy + bz * u)


C3_FACES = [0, 0, 0, 0, 0, 1]
C3_ALPHA = [0.0] * 5 + [1.0]


def c3_arrays(n, lo=(0, 0, 0), hi=(1, 1, 1)):
    return sample(n, lo, hi, c3_beta, c3_f, c3_u, lambda F, x, y, z: (1.0 + c3_beta(x, y, z)) * c3_u(x, y, z), C3_FACES)


# ---- linear patch with layered beta: u = 0.3 + 0.7 x - 0.4 y, beta_e random per element layer (z), f = 0,
#      Robin on x-, x+, y-, y+ (g_R = alpha_F u + beta_e du/dn_F, beta of the face element), Dirichlet z-, z+.
#      beta grad u = beta(z) (0.7, -0.4, 0) is divergence free, so u (a Q1 function) is the exact FE solution.
PATCH_FACES = [1, 1, 1, 1, 0, 0]
PATCH_ALPHA = [2.0, 0.5, 1.5, 3.0, 0.0, 0.0]
PATCH_DUDN = [-0.7, 0.7, 0.4, -0.4, 0.0, 0.0]


def patch_u(x, y, z):
    return 0.3 + 0.7 * x - 0.4 * y + 0.0 * z


def patch_arrays(n, layer_beta, lo=(0, 0, 0), hi=(1, 1, 1)):
    """layer_beta: n_z values (beta of element layer ez)."""
    lb = np.asarray(layer_beta, dtype=np.float64)
    hz = (hi[2] - lo[2]) / n[2]

    def beta_z(z):
        return lb[np.clip(np.floor((z - lo[2]) / hz).astype(np.int64), 0, n[2] - 1)]

    return sample(n, lo, hi, lambda x, y, z: beta_z(z), lambda x, y, z: 0.0 * x, patch_u,
                  lambda F, x, y, z: PATCH_ALPHA[F] * patch_u(x, y, z) + beta_z(z) * PATCH_DUDN[F], PATCH_FACES)


# ---- the same linear patch with alpha given at the face Gauss points (Eq. bvp's piecewise smooth alpha):
#      alpha_q random in [0, 3] at every Robin face Gauss point, g_R = alpha_q u + beta_e du/dn at the same points.
#      The Robin form int alpha u_h v and the load int g_R v use the same 2x2 Gauss points and alpha values, and
#      u is in Q1, so u is still the exact FE solution for ANY alpha_q >= 0.
def patch_alpha_q(n, seed=47, lo=(0, 0, 0), hi=(1, 1, 1)):
    """alpha at the 4 Gauss points of every face element, per face a block of 4 n_d1 n_d2 (gR's layout)."""
    blocks = []
    for F in range(6):
        d1, d2 = FACE_AXES[F]
        m = 4 * n[d1] * n[d2]
        blocks.append(3.0 * __import__("synth").counter_uniform(seed + F, m) if PATCH_FACES[F] == 1 else np.zeros(m))
    return np.concatenate(blocks)


def patch_arrays_alpha_q(n, layer_beta, aq, lo=(0, 0, 0), hi=(1, 1, 1)):
    """(beta_e, f_q, gD, gR, alpha_q) of the layered linear patch with alpha_q (patch_alpha_q) on the Robin faces."""
    b, fq, g, _ = patch_arrays(n, layer_beta, lo, hi)
    lb = np.asarray(layer_beta, dtype=np.float64)
    hz = (hi[2] - lo[2]) / n[2]
    blocks, off = [], 0
    for F in range(6):
        P = face_points(n, lo, hi, F)
        m = P[0].size
        a = aq[off:off + m].reshape(P[0].shape)
        off += m
        if PATCH_FACES[F] == 1:
            bz = lb[np.clip(np.floor((P[2] - lo[2]) / hz).astype(np.int64), 0, n[2] - 1)]
            blocks.append((a * patch_u(*P) + bz * PATCH_DUDN[F]).reshape(-1))
        else:
            blocks.append(np.zeros(m))
    return b, fq, g, np.concatenate(blocks), aq
