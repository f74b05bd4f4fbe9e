"""CPU oracle for ECMG_jcg (arXiv:1506.02983) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. The product path (paper_1506_02983_b200/) never imports it and shares no
code with it. The arithmetic lives in ecmg_oracle.cpp (plain C++, fp64, -ffp-contract=off);
this module only builds it (g++) and marshals numpy arrays through ctypes.

Parity status of each function is recorded in DESIGN.md ("Oracle pins"); every function here is
pinned by a `-m "not gpu"` test in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ecmg_oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

# problem ids / face kinds (interface numbers; the CUDA registry declares the same ids itself)
C1, C2, C3, C4, C5 = 1, 2, 3, 4, 5
P1, P2, P3 = 11, 12, 13
PATCH_TRILINEAR, PATCH_LAYERED, PATCH_ROBIN, CONST_F, PATCH_ROBIN_XY = 21, 22, 23, 24, 25
ARRAYS = 100   # caller data per level: beta_e, f at the Gauss points, g_D per node, g_R at the face Gauss points
DIRICHLET, ROBIN = 0, 1

NSTAT = 17
STAT_FIELDS = ["iterations", "rel_recur", "rel_true", "normb", "err_l2", "err_linf",
               "err_tilde_l2", "err_tilde_linf", "err_w_l2", "err_w_linf", "r_h",
               "t_setup", "t_exp", "t_solve", "t_rich", "status", "free_unknowns"]

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ -O2 -ffp-contract=off."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(LIB)
            dp, ip, vp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p
            L.orc_build_level.restype = vp
            L.orc_build_level.argtypes = [dp, dp, ip, C.c_int, dp, C.c_int, ip]
            L.orc_free_level.argtypes = [vp]
            L.orc_num_nodes.restype = C.c_long
            L.orc_num_nodes.argtypes = [vp]
            L.orc_get_matrix.argtypes = [vp, dp]
            L.orc_get_load.argtypes = [vp, dp]
            L.orc_get_rhs.restype = C.c_double
            L.orc_get_rhs.argtypes = [vp, dp]
            L.orc_get_dirichlet.argtypes = [vp, C.POINTER(C.c_ubyte), dp]
            L.orc_apply.argtypes = [vp, dp, dp]
            L.orc_jcg.restype = C.c_int
            L.orc_jcg.argtypes = [vp, dp, C.c_double, C.c_int, C.c_int, C.c_int, ip, dp, dp, dp]
            L.orc_dsolve.restype = C.c_int
            L.orc_dsolve.argtypes = [vp, dp]
            L.orc_exact.argtypes = [vp, dp]
            L.orc_exp_finite.restype = C.c_int
            L.orc_exp_finite.argtypes = [vp, dp, dp, dp, C.c_int]
            L.orc_exp_true.restype = C.c_int
            L.orc_exp_true.argtypes = [vp, dp, dp, dp]
            L.orc_norms.argtypes = [vp, dp, dp, dp]
            llp = C.POINTER(C.c_longlong)
            L.orc_rows.argtypes = [dp, dp, ip, C.c_int, dp, C.c_int, ip, llp, C.c_long, dp, dp, dp, dp]
            L.orc_rows.restype = C.c_int
            L.orc_exp_nodes.argtypes = [dp, dp, ip, C.c_int, dp, C.c_int, ip, C.c_int, dp, dp, llp, C.c_long, dp]
            L.orc_exp_nodes.restype = C.c_int
            L.orc_element_stiffness.argtypes = [dp, C.c_double, dp]
            L.orc_face_integrals.argtypes = [C.c_double, C.c_double, dp, dp, dp, dp]
            L.orc_serendipity_weights.argtypes = [C.c_double, C.c_double, C.c_double, dp]
            L.orc_ecmg.restype = C.c_int
            L.orc_ecmg.argtypes = [dp, dp, ip, C.c_int, C.c_int, dp, C.c_int, ip, C.c_double, C.c_int,
                                   C.c_int, C.c_int, dp, dp, dp, dp]
            L.orc_build_level_arrays.restype = vp
            L.orc_build_level_arrays.argtypes = [dp, dp, ip, ip, dp, dp, dp, dp, dp, dp]
            L.orc_ecmg_arrays.restype = C.c_int
            L.orc_ecmg_arrays.argtypes = [dp, dp, ip, C.c_int, dp, ip, C.POINTER(dp), C.c_int, C.c_double, C.c_int,
                                          C.c_int, C.c_int, dp, dp, dp, dp]
            L.orc_ecmg_fixed_arrays.restype = C.c_int
            L.orc_ecmg_fixed_arrays.argtypes = [dp, dp, ip, C.c_int, dp, ip, C.POINTER(dp), C.c_int, C.c_int,
                                                C.c_double, C.c_int, C.c_int, dp, dp, dp, dp]
            L.orc_ecmg_fixed.restype = C.c_int
            L.orc_ecmg_fixed.argtypes = [dp, dp, ip, C.c_int, C.c_int, dp, C.c_int, ip, C.c_int, C.c_double,
                                         C.c_int, C.c_int, dp, dp, dp, dp]
            L.orc_set_threads.restype = C.c_int
            L.orc_set_threads.argtypes = [C.c_int]
            L.orc_get_threads.restype = C.c_int
            L.orc_max_threads.restype = C.c_int
            _lib = L
    return _lib


def set_threads(t: int) -> int:
    """Threads of the oracle's row loops (1 = serial). Results are bitwise the same for every t
    (tests/test_oracle_threads.py); only the wall time changes. Returns the previous value."""
    prev = lib().orc_get_threads()
    if lib().orc_set_threads(int(t)) != 0:
        raise ValueError(f"oracle: bad thread count {t}")
    return prev


def max_threads() -> int:
    """Host processors available to the oracle (omp_get_num_procs)."""
    return int(lib().orc_max_threads())


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def default_faces(problem_id: int):
    f = [DIRICHLET] * 6
    if problem_id in (C3, PATCH_ROBIN):
        f[5] = ROBIN
    elif problem_id == P1:
        f[1] = f[3] = f[5] = ROBIN
    elif problem_id == P2:
        f[1] = f[3] = ROBIN
    elif problem_id == PATCH_ROBIN_XY:
        f[0] = f[1] = f[2] = f[3] = ROBIN
    return f


class Level:
    """One assembled grid level (explicit 27-band matrix, lifted RHS, node classes)."""

    def __init__(self, n_cells, problem_id, params=None, lo=(0, 0, 0), hi=(1, 1, 1), faces=None):
        L = lib()
        self.n = tuple(int(v) for v in n_cells)
        self.shape = (self.n[2] + 1, self.n[1] + 1, self.n[0] + 1)
        self.N = self.shape[0] * self.shape[1] * self.shape[2]
        self.problem_id = problem_id
        self.params = _f64(params if params is not None else np.zeros(1))
        self.faces = np.array(faces if faces is not None else default_faces(problem_id), dtype=np.int32)
        self.lo, self.hi = _f64(lo), _f64(hi)
        n = np.array(self.n, dtype=np.int32)
        self._h = L.orc_build_level(_d(self.lo), _d(self.hi), _i(n), problem_id, _d(self.params),
                                    int(self.params.size if params is not None else 0), _i(self.faces))
        if not self._h:
            raise ValueError("oracle: invalid level / problem")

    @classmethod
    def from_arrays(cls, n_cells, faces, alpha, beta_e=None, f_q=None, gD=None, gR=None, lo=(0, 0, 0), hi=(1, 1, 1),
                    alpha_q=None):
        """A level of the ARRAYS problem: beta_e[n_x n_y n_z] (x fastest), f_q[8 per element] (Gauss point
        q = q_x + 2 q_y + 4 q_z, bit set = +1/sqrt(3)), gD[(n_x+1)(n_y+1)(n_z+1)], gR[per face x-..z+ a block of
        4 n_d1 n_d2: 4 (e1 + n_d1 e2) + q], alpha[6]; None = beta 1 / f 0 / g_D 0 / g_R 0. alpha_q: alpha at the
        face Gauss points in gR's layout (Eq. bvp's piecewise smooth alpha), None = alpha[F] per face."""
        self = cls.__new__(cls)
        L = lib()
        self.n = tuple(int(v) for v in n_cells)
        self.shape = (self.n[2] + 1, self.n[1] + 1, self.n[0] + 1)
        self.N = self.shape[0] * self.shape[1] * self.shape[2]
        self.problem_id = ARRAYS
        self.params = _f64(alpha)
        self.faces = np.array(faces, dtype=np.int32)
        self.lo, self.hi = _f64(lo), _f64(hi)
        self._arrays = [None if a is None else _f64(a).reshape(-1) for a in (beta_e, f_q, gD, gR, alpha_q)]
        n = np.array(self.n, dtype=np.int32)
        ptr = [_d(a) if a is not None else None for a in self._arrays]
        self._h = L.orc_build_level_arrays(_d(self.lo), _d(self.hi), _i(n), _i(self.faces), _d(self.params), *ptr)
        if not self._h:
            raise ValueError("oracle: invalid ARRAYS level")
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_free_level(h)
            self._h = None

    def matrix(self):
        A = np.empty(self.N * 27)
        lib().orc_get_matrix(self._h, _d(A))
        return A.reshape(self.N, 27)

    def load(self):
        F = np.empty(self.N)
        lib().orc_get_load(self._h, _d(F))
        return F

    def rhs(self):
        b = np.empty(self.N)
        nb = lib().orc_get_rhs(self._h, _d(b))
        return b, nb

    def dirichlet(self):
        m = np.empty(self.N, dtype=np.uint8)
        g = np.empty(self.N)
        lib().orc_get_dirichlet(self._h, m.ctypes.data_as(C.POINTER(C.c_ubyte)), _d(g))
        return m.astype(bool), g

    def apply(self, p):
        p = _f64(p)
        q = np.empty(self.N)
        lib().orc_apply(self._h, _d(p), _d(q))
        return q

    def jcg(self, x0, eps, max_iter, precond=True, dot_reverse=False):
        """Textbook JCG / CG. dot_reverse sums the dot products in reverse node order: only for
        measuring the oracle's own rounding-order spread."""
        x = _f64(x0).copy()
        it, rr, rt, nb = C.c_int(), C.c_double(), C.c_double(), C.c_double()
        st = lib().orc_jcg(self._h, _d(x), float(eps), int(max_iter), 1 if precond else 0, 1 if dot_reverse else 0,
                           C.byref(it), C.byref(rr), C.byref(rt), C.byref(nb))
        return x, dict(status=st, iterations=it.value, rel_recur=rr.value, rel_true=rt.value, normb=nb.value)

    def dsolve(self):
        x = np.zeros(self.N)
        st = lib().orc_dsolve(self._h, _d(x))
        if st != 0:
            raise RuntimeError(f"oracle dsolve failed: {st}")
        return x

    def exact(self):
        u = np.empty(self.N)
        lib().orc_exact(self._h, _d(u))
        return u

    def exp_finite(self, u2h, u4h, variant=0):
        """variant 0: 20-node Serendipity; 1: Remark 2's 27-node Lagrange."""
        w = np.empty(self.N)
        st = lib().orc_exp_finite(self._h, _d(_f64(u2h)), _d(_f64(u4h)), _d(w), int(variant))
        if st != 0:
            raise ValueError(f"oracle exp_finite: {st}")
        return w

    def exp_true(self, uh, u2h):
        ut = np.empty(self.N)
        st = lib().orc_exp_true(self._h, _d(_f64(uh)), _d(_f64(u2h)), _d(ut))
        if st != 0:
            raise ValueError(f"oracle exp_true: {st}")
        return ut

    def norms(self, e):
        l2, li = C.c_double(), C.c_double()
        lib().orc_norms(self._h, _d(_f64(e)), C.byref(l2), C.byref(li))
        return l2.value, li.value


def element_stiffness(h, beta=1.0):
    K = np.empty(64)
    lib().orc_element_stiffness(_d(_f64(h)), float(beta), _d(K))
    return K.reshape(8, 8)


def face_integrals(h1, h2, alpha_q, g_q):
    M = np.empty(16)
    G = np.empty(4)
    lib().orc_face_integrals(float(h1), float(h2), _d(_f64(alpha_q)), _d(_f64(g_q)), _d(M), _d(G))
    return M.reshape(4, 4), G


SEED_LABELS = [1, 3, 5, 11, 15, 21, 23, 25, 51, 55, 71, 75, 101, 103, 105, 111, 115, 121, 123, 125]


def serendipity_weights(xi, eta, zeta):
    w = np.empty(20)
    lib().orc_serendipity_weights(float(xi), float(eta), float(zeta), _d(w))
    return w


def ecmg(n0, levels, problem_id, eps, params=None, lo=(0, 0, 0), hi=(1, 1, 1), faces=None,
         max_iter=100000, precond=True, want_w=False, exp_variant=0):
    """Alg. 4. Returns (status, stats[levels, NSTAT], u_fine, ut_fine[, w_fine])."""
    n0 = np.array([n0] * 3 if np.isscalar(n0) else list(n0), dtype=np.int32)
    nf = n0 * (1 << (levels - 1))
    N = int(np.prod(nf + 1))
    stats = np.empty(levels * NSTAT)
    u = np.empty(N)
    ut = np.empty(N)
    w = np.empty(N) if want_w else None
    prm = _f64(params if params is not None else np.zeros(1))
    fc = np.array(faces if faces is not None else default_faces(problem_id), dtype=np.int32)
    st = lib().orc_ecmg(_d(_f64(lo)), _d(_f64(hi)), _i(n0), int(levels), int(problem_id), _d(prm),
                        int(prm.size if params is not None else 0), _i(fc), float(eps), int(max_iter),
                        1 if precond else 0, int(exp_variant), _d(stats), _d(u), _d(ut),
                        _d(w) if w is not None else None)
    stats = stats.reshape(levels, NSTAT)
    if want_w:
        return st, stats, u, ut, w
    return st, stats, u, ut


def _level_ptrs(level_arrays):
    """The oracle's level-array list: (beta_e, f_q, gD, gR) of every level, then alpha_q of every level when the
    tuples carry a fifth entry (n_level_arrays = 4 L or 5 L)."""
    with_alpha = any(len(lv) > 4 for lv in level_arrays)
    arrs = [a for lv in level_arrays for a in lv[:4]]
    if with_alpha:
        arrs += [lv[4] if len(lv) > 4 else None for lv in level_arrays]
    keep = [None if a is None else _f64(a).reshape(-1) for a in arrs]
    return keep, len(keep)


def ecmg_arrays(n0, levels, faces, alpha, level_arrays, eps, lo=(0, 0, 0), hi=(1, 1, 1), max_iter=100000,
                precond=True, want_w=False, exp_variant=0):
    """Alg. 4 on ARRAYS data: level_arrays[k] = (beta_e, f_q, gD, gR[, alpha_q]) of level k (layouts:
    Level.from_arrays); alpha_q given on every level or on none."""
    n0 = np.array([n0] * 3 if np.isscalar(n0) else list(n0), dtype=np.int32)
    nf = n0 * (1 << (levels - 1))
    N = int(np.prod(nf + 1))
    stats = np.empty(levels * NSTAT)
    u, ut = np.empty(N), np.empty(N)
    w = np.empty(N) if want_w else None
    keep, nla = _level_ptrs(level_arrays)
    ptrs = (C.POINTER(C.c_double) * len(keep))(*[_d(a) if a is not None else None for a in keep])
    fc = np.array(faces, dtype=np.int32)
    st = lib().orc_ecmg_arrays(_d(_f64(lo)), _d(_f64(hi)), _i(n0), int(levels), _d(_f64(alpha)), _i(fc), ptrs, nla,
                               float(eps), int(max_iter), 1 if precond else 0, int(exp_variant), _d(stats), _d(u),
                               _d(ut), _d(w) if w is not None else None)
    del keep
    stats = stats.reshape(levels, NSTAT)
    if want_w:
        return st, stats, u, ut, w
    return st, stats, u, ut


def ecmg_fixed_arrays(n0, levels, faces, alpha, level_arrays, m_L, ratio, lo=(0, 0, 0), hi=(1, 1, 1), precond=False,
                      exp_variant=0):
    """Alg. 3 on ARRAYS data (level_arrays as in ecmg_arrays)."""
    n0 = np.array([n0] * 3 if np.isscalar(n0) else list(n0), dtype=np.int32)
    N = int(np.prod(n0 * (1 << (levels - 1)) + 1))
    stats = np.empty(levels * NSTAT)
    u, ut = np.empty(N), np.empty(N)
    keep, nla = _level_ptrs(level_arrays)
    ptrs = (C.POINTER(C.c_double) * len(keep))(*[_d(a) if a is not None else None for a in keep])
    st = lib().orc_ecmg_fixed_arrays(_d(_f64(lo)), _d(_f64(hi)), _i(n0), int(levels), _d(_f64(alpha)),
                                     _i(np.array(faces, dtype=np.int32)), ptrs, nla, int(m_L), float(ratio),
                                     1 if precond else 0, int(exp_variant), _d(stats), _d(u), _d(ut), None)
    del keep
    return st, stats.reshape(levels, NSTAT), u, ut


def ecmg_fixed(n0, levels, problem_id, m_L, ratio, params=None, lo=(0, 0, 0), hi=(1, 1, 1), faces=None,
               precond=False, exp_variant=0, want_w=False):
    """Alg. 3: fixed m_j = ceil(m_L ratio^(L-j)) CG iterations on the j-th ECMG level."""
    n0 = np.array([n0] * 3 if np.isscalar(n0) else list(n0), dtype=np.int32)
    nf = n0 * (1 << (levels - 1))
    N = int(np.prod(nf + 1))
    stats = np.empty(levels * NSTAT)
    u, ut = np.empty(N), np.empty(N)
    w = np.empty(N) if want_w else None
    prm = _f64(params if params is not None else np.zeros(1))
    fc = np.array(faces if faces is not None else default_faces(problem_id), dtype=np.int32)
    st = lib().orc_ecmg_fixed(_d(_f64(lo)), _d(_f64(hi)), _i(n0), int(levels), int(problem_id), _d(prm),
                              int(prm.size if params is not None else 0), _i(fc), int(m_L), float(ratio),
                              1 if precond else 0, int(exp_variant), _d(stats), _d(u), _d(ut),
                              _d(w) if w is not None else None)
    stats = stats.reshape(levels, NSTAT)
    return (st, stats, u, ut, w) if want_w else (st, stats, u, ut)


# ---- sampled evaluation without assembling the level (parity at full size) -------------------------
def _nodes(nodes):
    a = np.ascontiguousarray(np.asarray(nodes, dtype=np.int64).reshape(-1, 3))
    return a, a.ctypes.data_as(C.POINTER(C.c_longlong))


def rows(n_cells, problem_id, nodes, p=None, params=None, lo=(0, 0, 0), hi=(1, 1, 1), faces=None, diag=False):
    """(A_ff p)_i and the lifted b_f,i at the given (ix, iy, iz) nodes, each row accumulated from the
    element (and Robin face) matrices around the node in build_level's order; with diag=True also A_ii."""
    nd, ndp = _nodes(nodes)
    n = np.array([int(v) for v in n_cells], dtype=np.int32)
    prm = _f64(params if params is not None else np.zeros(1))
    fc = np.array(faces if faces is not None else default_faces(problem_id), dtype=np.int32)
    q = np.empty(len(nd))
    b = np.empty(len(nd))
    pp = _f64(p) if p is not None else None
    dg = np.empty(len(nd)) if diag else None
    st = lib().orc_rows(_d(_f64(lo)), _d(_f64(hi)), _i(n), problem_id, _d(prm),
                        int(prm.size if params is not None else 0), _i(fc), ndp, len(nd),
                        _d(pp) if pp is not None else None, _d(q) if pp is not None else None, _d(b),
                        _d(dg) if diag else None)
    if st != 0:
        raise ValueError(f"oracle rows: {st}")
    if diag:
        return (q if pp is not None else None), b, dg
    return (q if pp is not None else None), b


def exp_nodes(n_cells, problem_id, which, a, c, nodes, params=None, lo=(0, 0, 0), hi=(1, 1, 1), faces=None):
    """which 0: EXP_finite (Serendipity), 1: EXP_finite (Remark 2 Lagrange), 2: EXP_true, at the given
    fine nodes; a, c = (u_2h, u_4h) or (u_h, u_2h) as full nodal vectors."""
    nd, ndp = _nodes(nodes)
    n = np.array([int(v) for v in n_cells], dtype=np.int32)
    prm = _f64(params if params is not None else np.zeros(1))
    fc = np.array(faces if faces is not None else default_faces(problem_id), dtype=np.int32)
    out = np.empty(len(nd))
    st = lib().orc_exp_nodes(_d(_f64(lo)), _d(_f64(hi)), _i(n), problem_id, _d(prm),
                             int(prm.size if params is not None else 0), _i(fc), int(which), _d(_f64(a)),
                             _d(_f64(c)), ndp, len(nd), _d(out))
    if st != 0:
        raise ValueError(f"oracle exp_nodes: {st}")
    return out
