"""ctypes binding of libecmg (include/ecmg.h): argument marshalling only.

Every step of the hot path runs in libecmg's CUDA kernels; this module converts torch tensors
to raw device pointers, C structs and status codes. There is no CPU fallback: if libecmg.so is
missing or fails to load, every call raises.

Names follow the C ABI: create_grid, set_coeffs, solve_level, prolongate_extrapolate,
richardson, run, apply_operator, level_rhs, level_shape, set_option, last_jcg_timing,
destroy_grid, strerror. `Grid` is a small RAII wrapper over them.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libecmg.so")

OK, EINVAL, ENOMEM, ENOTCONV, EBREAKDOWN, EDIAG, EMISMATCH, ECUDA, ENCCL = 0, -1, -2, -3, -4, -5, -6, -7, -8
DIRICHLET, ROBIN = 0, 1
PROB = dict(C1=1, C2=2, C3=3, C4=4, C5=5, P1=11, P2=12, P3=13,
            PATCH_TRILINEAR=21, PATCH_LAYERED=22, PATCH_ROBIN=23, CONST_F=24, PATCH_ROBIN_XY=25,
            ARRAYS=100)
OPT_EXP_VARIANT, OPT_PRECOND, OPT_ZCHUNK, OPT_KERNEL, OPT_GRAPH, OPT_VIRTUAL_SLABS, OPT_PERSISTENT, OPT_PDL = 1, 2, 3, 4, 5, 6, 7, 8
OPT_FUSED_HALO = 9
OPT_SETUP_AHEAD = 10
OPT_SETUP_CTAS = 11
OPT_EXP_KERNEL = 12
OPT_CTA_SOLVE = 13
OPT_PERS_TMA = 14
OPT_BETA_FLY = 15
OPT_SLAB_HYBRID = 16
OPT_UNFUSED = 17
OPT_SHARD_MIN = 18
OPT_XDEFER = 19
OPT_RHS_SYM = 20
OPT_RICH_FUSED = 21
OPT_P0_INIT = 22

EXPORTS = ["ecmg_create_grid", "ecmg_set_coeffs", "ecmg_set_option", "ecmg_solve_level",
           "ecmg_prolongate_extrapolate", "ecmg_richardson", "ecmg_run", "ecmg_run_fixed", "ecmg_apply_operator",
           "ecmg_level_rhs", "ecmg_level_shape", "ecmg_last_jcg_timing", "ecmg_kernel_launches",
           "ecmg_slab_partition", "ecmg_nccl_unique_id", "ecmg_destroy_grid", "ecmg_strerror"]


class ecmg_box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3)]


class ecmg_dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("nccl_id", C.c_ubyte * 128)]


class ecmg_problem(C.Structure):
    _fields_ = [("face", C.c_int * 6), ("problem_id", C.c_int), ("params", C.POINTER(C.c_double)),
                ("n_params", C.c_int), ("level_arrays", C.POINTER(C.POINTER(C.c_double))),
                ("n_level_arrays", C.c_int)]


class ecmg_stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("rel_res_recur", C.c_double), ("rel_res_true", C.c_double),
                ("norm_b", C.c_double), ("converged", C.c_int), ("status", C.c_int),
                ("ms_setup", C.c_double), ("ms_exp", C.c_double), ("ms_solve", C.c_double),
                ("ms_rich", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class EcmgError(RuntimeError):
    def __init__(self, status, where):
        super().__init__(f"{where}: {strerror(status)} ({status})")
        self.status = status


_lib = None


def lib():
    """Load libecmg.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libecmg.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.ecmg_create_grid.argtypes = [C.POINTER(ecmg_box), ip, C.c_int, C.POINTER(ecmg_dist), vp, C.POINTER(vp)]
        L.ecmg_set_coeffs.argtypes = [vp, C.POINTER(ecmg_problem)]
        L.ecmg_set_option.argtypes = [vp, C.c_int, C.c_int]
        L.ecmg_solve_level.argtypes = [vp, C.c_int, C.c_double, C.c_int, vp, C.POINTER(ecmg_stats)]
        L.ecmg_prolongate_extrapolate.argtypes = [vp, C.c_int, vp, vp, vp]
        L.ecmg_richardson.argtypes = [vp, C.c_int, vp, vp, vp]
        L.ecmg_run.argtypes = [vp, C.c_double, C.POINTER(ecmg_stats), vp, vp]
        L.ecmg_run_fixed.argtypes = [vp, C.c_int, C.c_double, C.POINTER(ecmg_stats), vp, vp]
        L.ecmg_apply_operator.argtypes = [vp, C.c_int, vp, vp]
        L.ecmg_level_rhs.argtypes = [vp, C.c_int, vp, dp]
        L.ecmg_level_shape.argtypes = [vp, C.c_int, ip, C.POINTER(C.c_longlong), ip, ip]
        L.ecmg_last_jcg_timing.argtypes = [vp, dp, ip, C.POINTER(C.c_longlong)]
        L.ecmg_kernel_launches.argtypes = []
        L.ecmg_slab_partition.argtypes = [C.c_int, C.c_int, C.c_int, ip, ip]
        L.ecmg_nccl_unique_id.argtypes = [C.POINTER(C.c_ubyte)]
        L.ecmg_destroy_grid.argtypes = [vp]
        L.ecmg_strerror.argtypes = [C.c_int]
        L.ecmg_strerror.restype = C.c_char_p
        for name in EXPORTS:
            if name not in ("ecmg_strerror", "ecmg_kernel_launches"):
                getattr(L, name).restype = C.c_int
        L.ecmg_kernel_launches.restype = C.c_longlong
        _lib = L
    return _lib


def strerror(status: int) -> str:
    return lib().ecmg_strerror(int(status)).decode()


def _ptr(t):
    """Raw pointer of a torch tensor (device or host) or numpy array."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if t.dtype != __import__("torch").float64 or not t.is_contiguous():
            raise TypeError("libecmg takes contiguous float64 tensors")
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


# ---- C-ABI-named functions (return the status code, never raise on solver statuses) ------------

def create_grid(lo, hi, coarsest_cells, num_levels, stream=None, dist=None):
    box = ecmg_box((C.c_double * 3)(*lo), (C.c_double * 3)(*hi))
    cc = (C.c_int * 3)(*coarsest_cells)
    out = C.c_void_p()
    st = lib().ecmg_create_grid(C.byref(box), cc, int(num_levels), C.byref(dist) if dist else None,
                                C.c_void_p(stream) if stream else None, C.byref(out))
    return st, out


def set_coeffs(grid, problem_id, faces, params=None, level_arrays=None):
    """level_arrays (ECMG_PROB_ARRAYS): 4 device arrays (or None) per level, flattened in level order, optionally
    followed by one alpha_q array (or None) per level (5 L in all); the
    library keeps the pointers, the caller keeps the arrays alive (include/ecmg.h)."""
    pr = ecmg_problem()
    for i, f in enumerate(faces):
        pr.face[i] = int(f)
    pr.problem_id = int(problem_id)
    keep = None
    if params is not None:
        keep = (C.c_double * len(params))(*[float(v) for v in params])
        pr.params = C.cast(keep, C.POINTER(C.c_double))
        pr.n_params = len(params)
    if level_arrays is not None:
        dp = C.POINTER(C.c_double)
        arr = (dp * len(level_arrays))(*[C.cast(_ptr(a), dp) if a is not None else dp()
                                         for a in level_arrays])
        pr.level_arrays = C.cast(arr, C.POINTER(dp))
        pr.n_level_arrays = len(level_arrays)
    return lib().ecmg_set_coeffs(grid, C.byref(pr))


def set_option(grid, option, value):
    return lib().ecmg_set_option(grid, int(option), int(value))


def solve_level(grid, level, eps, max_iter, u):
    st = ecmg_stats()
    s = lib().ecmg_solve_level(grid, int(level), float(eps), int(max_iter), _ptr(u), C.byref(st))
    return s, st


def prolongate_extrapolate(grid, level, u2h, u4h, w):
    return lib().ecmg_prolongate_extrapolate(grid, int(level), _ptr(u2h), _ptr(u4h), _ptr(w))


def richardson(grid, level, uh, u2h, ut):
    return lib().ecmg_richardson(grid, int(level), _ptr(uh), _ptr(u2h), _ptr(ut))


def run(grid, eps, num_levels, u_fine, ut_fine=None):
    stats = (ecmg_stats * num_levels)()
    s = lib().ecmg_run(grid, float(eps), stats, _ptr(u_fine), _ptr(ut_fine))
    return s, [stats[k] for k in range(num_levels)]


def run_fixed(grid, m_L, ratio, num_levels, u_fine, ut_fine=None):
    stats = (ecmg_stats * num_levels)()
    s = lib().ecmg_run_fixed(grid, int(m_L), float(ratio), stats, _ptr(u_fine), _ptr(ut_fine))
    return s, [stats[k] for k in range(num_levels)]


def apply_operator(grid, level, p, q):
    return lib().ecmg_apply_operator(grid, int(level), _ptr(p), _ptr(q))


def level_rhs(grid, level, b):
    nb = C.c_double()
    s = lib().ecmg_level_rhs(grid, int(level), _ptr(b), C.byref(nb))
    return s, nb.value


def level_shape(grid, level):
    n = (C.c_int * 3)()
    nodes = C.c_longlong()
    zlo, zhi = C.c_int(), C.c_int()
    s = lib().ecmg_level_shape(grid, int(level), n, C.byref(nodes), C.byref(zlo), C.byref(zhi))
    return s, tuple(n), nodes.value, zlo.value, zhi.value


def last_jcg_timing(grid):
    ms, it, nf = C.c_double(), C.c_int(), C.c_longlong()
    s = lib().ecmg_last_jcg_timing(grid, C.byref(ms), C.byref(it), C.byref(nf))
    return s, ms.value, it.value, nf.value


def kernel_launches():
    return int(lib().ecmg_kernel_launches())


def slab_partition(n_cells_z, nranks, rank):
    """(sharded, z_lo, z_hi) of rank's node planes [z_lo, z_hi) on a level with n_cells_z cells."""
    lo, hi = C.c_int(), C.c_int()
    s = lib().ecmg_slab_partition(int(n_cells_z), int(nranks), int(rank), C.byref(lo), C.byref(hi))
    if s < 0:
        raise EcmgError(s, "ecmg_slab_partition")
    return bool(s), lo.value, hi.value


def nccl_unique_id():
    buf = (C.c_ubyte * 128)()
    s = lib().ecmg_nccl_unique_id(buf)
    if s != OK:
        raise EcmgError(s, "ecmg_nccl_unique_id")
    return bytes(buf)


def make_dist(rank, nranks, nccl_id: bytes):
    d = ecmg_dist()
    d.rank, d.nranks = int(rank), int(nranks)
    for i, b in enumerate(nccl_id[:128]):
        d.nccl_id[i] = b
    return d


def destroy_grid(grid):
    return lib().ecmg_destroy_grid(grid)


def default_faces(problem_id: int):
    f = [DIRICHLET] * 6
    if problem_id in (PROB["C3"], PROB["PATCH_ROBIN"]):
        f[5] = ROBIN
    elif problem_id == PROB["P1"]:
        f[1] = f[3] = f[5] = ROBIN
    elif problem_id == PROB["P2"]:
        f[1] = f[3] = ROBIN
    elif problem_id == PROB["PATCH_ROBIN_XY"]:
        f[0] = f[1] = f[2] = f[3] = ROBIN
    return f


class Grid:
    """Owning wrapper: Grid(coarsest, levels, problem_id, params) on the current torch stream."""

    def __init__(self, coarsest, num_levels, problem_id, params=None, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
                 stream=None, exp_variant=0, precond=True, dist=None, faces=None, level_arrays=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        coarsest = [coarsest] * 3 if isinstance(coarsest, int) else list(coarsest)
        self.coarsest, self.L, self.problem_id = coarsest, num_levels, problem_id
        self.device = torch.cuda.current_device()
        st, self.h = create_grid(lo, hi, coarsest, num_levels, stream, dist)
        if st != OK:
            raise EcmgError(st, "ecmg_create_grid")
        # ARRAYS: level_arrays[k] = (beta_e, f_q, gD, gR[, alpha_q]) device float64 tensors (or None), kept alive
        # here; the ABI order is the 4 of every level, then alpha_q of every level (n_level_arrays = 5 L)
        self._arrays = None
        if level_arrays is not None:
            self._arrays = [a for lv in level_arrays for a in lv[:4]]
            if any(len(lv) > 4 for lv in level_arrays):
                self._arrays += [lv[4] if len(lv) > 4 else None for lv in level_arrays]
        self._check(set_coeffs(self.h, problem_id, faces if faces is not None else default_faces(problem_id), params,
                               self._arrays), "ecmg_set_coeffs")
        self._check(set_option(self.h, OPT_EXP_VARIANT, exp_variant), "ecmg_set_option")
        self._check(set_option(self.h, OPT_PRECOND, 1 if precond else 0), "ecmg_set_option")

    @staticmethod
    def _check(st, where, allow=(OK,)):
        if st not in allow:
            raise EcmgError(st, where)
        return st

    def shape(self, level):
        _, n, nodes, _, _ = level_shape(self.h, level)
        return n, nodes

    def _vec(self, t, level, where, host_ok=False):
        """Check a caller vector before its raw pointer crosses the ABI: float64, contiguous, at least the
        level's node count, and on this grid's device (or, where the ABI allows it, in host memory)."""
        if t is None:
            return None
        if not hasattr(t, "data_ptr"):
            raise TypeError(f"{where}: expected a torch tensor")
        if str(t.dtype) != "torch.float64" or not t.is_contiguous():
            raise TypeError(f"{where}: libecmg takes contiguous float64 tensors")
        _, nodes = self.shape(level)
        if t.numel() < nodes:
            raise ValueError(f"{where}: tensor has {t.numel()} elements, level {level} has {nodes} nodes")
        if t.is_cuda:
            if t.device.index != self.device:
                raise ValueError(f"{where}: tensor on cuda:{t.device.index}, grid on cuda:{self.device}")
        elif not host_ok:
            raise ValueError(f"{where}: a device tensor is required")
        return t

    def new_vec(self, level, device="cuda"):
        import torch
        n, nodes = self.shape(level)
        return torch.zeros(nodes, dtype=torch.float64, device=device)

    def solve_level(self, level, eps, max_iter, u):
        self._vec(u, level, "solve_level(u)")
        st, stats = solve_level(self.h, level, eps, max_iter, u)
        self._check(st, "ecmg_solve_level", allow=(OK, ENOTCONV))
        return st, stats.as_dict()

    def prolongate_extrapolate(self, level, u2h, u4h, w):
        self._vec(u2h, level - 1, "prolongate_extrapolate(u2h)")
        self._vec(u4h, level - 2, "prolongate_extrapolate(u4h)")
        self._vec(w, level, "prolongate_extrapolate(w)")
        self._check(prolongate_extrapolate(self.h, level, u2h, u4h, w), "ecmg_prolongate_extrapolate")

    def richardson(self, level, uh, u2h, ut):
        self._vec(uh, level, "richardson(uh)")
        self._vec(u2h, level - 1, "richardson(u2h)")
        self._vec(ut, level, "richardson(ut)")
        self._check(richardson(self.h, level, uh, u2h, ut), "ecmg_richardson")

    def run(self, eps, u_fine, ut_fine=None):
        self._vec(u_fine, self.L - 1, "run(u_fine)", host_ok=True)
        self._vec(ut_fine, self.L - 1, "run(ut_fine)", host_ok=True)
        st, stats = run(self.h, eps, self.L, u_fine, ut_fine)
        self._check(st, "ecmg_run", allow=(OK, ENOTCONV))
        return st, [s.as_dict() for s in stats]

    def run_fixed(self, m_L, ratio, u_fine, ut_fine=None):
        self._vec(u_fine, self.L - 1, "run_fixed(u_fine)", host_ok=True)
        self._vec(ut_fine, self.L - 1, "run_fixed(ut_fine)", host_ok=True)
        st, stats = run_fixed(self.h, m_L, ratio, self.L, u_fine, ut_fine)
        self._check(st, "ecmg_run_fixed")
        return st, [s.as_dict() for s in stats]

    def apply_operator(self, level, p, q):
        self._vec(p, level, "apply_operator(p)")
        self._vec(q, level, "apply_operator(q)")
        self._check(apply_operator(self.h, level, p, q), "ecmg_apply_operator")

    def level_rhs(self, level, b):
        self._vec(b, level, "level_rhs(b)")
        st, nb = level_rhs(self.h, level, b)
        self._check(st, "ecmg_level_rhs")
        return nb

    def set_option(self, option, value):
        self._check(set_option(self.h, option, value), "ecmg_set_option")

    def last_jcg_timing(self):
        _, ms, it, nf = last_jcg_timing(self.h)
        return ms, it, nf

    def close(self):
        if getattr(self, "h", None):
            destroy_grid(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
