"""Seeded synthetic inputs shared by the oracle tests, the GPU tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no stencil, no extrapolation, no solver).
It only draws numbers: the splitmix64 counter generator, seeded random nodal vectors for
parity tests (SURVEY.md §8d "Parity inputs (T1)"), and the realised C5 "layered geology"
geometry (SURVEY.md §8c A18 / §8d "C5 recipe"). Both sides receive the numbers it draws as
plain input arrays, so neither the oracle nor the CUDA path imports the other.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class SplitMix64:
    """Sequential splitmix64: state += GOLDEN; return mix(state). Draw u = (next >> 11) * 2^-53."""

    def __init__(self, seed: int = 0):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        return _mix(self.state)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = (self.next_u64() >> 11) * (2.0 ** -53)
        return lo + (hi - lo) * u


def _mix_vec(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, count: int) -> np.ndarray:
    """u_i = (mix(seed*2^40 + i + GOLDEN) >> 11) * 2^-53 in [0,1), i = 0..count-1 (counter based)."""
    base = np.uint64((seed << 40) & MASK64)
    with np.errstate(over="ignore"):
        c = base + np.arange(count, dtype=np.uint64) + np.uint64(GOLDEN)
    z = _mix_vec(c)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def random_nodal(seed: int, n_cells, free_lo=None, free_hi=None) -> np.ndarray:
    """Seeded vector on the (nx+1)(ny+1)(nz+1) nodes, x fastest: x_i = 2u_i - 1 on the free box,
    0 elsewhere (0 on Dirichlet nodes). free_lo/free_hi are inclusive node
    index bounds per axis; None means all nodes."""
    nx, ny, nz = (int(v) for v in n_cells)
    shape = (nz + 1, ny + 1, nx + 1)
    v = (2.0 * counter_uniform(seed, shape[0] * shape[1] * shape[2]) - 1.0).reshape(shape)
    if free_lo is not None:
        mask = np.zeros(shape, dtype=bool)
        lo, hi = free_lo, free_hi
        mask[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1] = True
        v = np.where(mask, v, 0.0)
    return np.ascontiguousarray(v.reshape(-1))


# ---------------------------------------------------------------------------------------------
# C5 "layered geology" geometry (BASELINE.json configs[4]; SURVEY.md §8d C5 recipe)
# params layout (48 doubles), read identically by the oracle and by the CUDA problem registry:
#   [0:7]   7 sorted interface heights z_1 < ... < z_7 (8 layers)
#   [7:15]  8 layer beta values
#   [15:43] 4 boxes x (cx, cy, cz, sx, sy, sz, beta)   (centre, half-widths, value)
#   [43:46] source point x0
#   [46]    sigma (0.05)
#   [47]    source amplitude (1.0, unnormalised)
# ---------------------------------------------------------------------------------------------
C5_NPARAMS = 48


def c5_geometry(seed: int = 0) -> np.ndarray:
    g = SplitMix64(seed)
    heights = sorted(g.uniform() for _ in range(7))
    layer_beta = [10.0 ** (2.0 * g.uniform() - 1.0) for _ in range(8)]
    boxes = []
    for _ in range(4):
        c = [g.uniform(0.15, 0.85) for _ in range(3)]
        s = [g.uniform(0.05, 0.20) for _ in range(3)]
        b = 10.0 ** (2.0 * g.uniform() - 1.0)
        boxes += c + s + [b]
    x0 = [g.uniform(0.25, 0.75) for _ in range(3)]
    p = np.array(heights + layer_beta + boxes + x0 + [0.05, 1.0], dtype=np.float64)
    assert p.size == C5_NPARAMS
    return p


def layered_only(seed: int = 0) -> np.ndarray:
    """The C5 layer set with no boxes (for the layered-beta patch test)."""
    return c5_geometry(seed)[:15].copy()


def face_gauss_count(n_cells) -> int:
    """Length of a g_R array of the ARRAYS problem: 4 Gauss points per face element, all six faces."""
    nx, ny, nz = (int(v) for v in n_cells)
    return 4 * 2 * (ny * nz + nx * nz + nx * ny)


def random_problem_arrays(seed: int, n_cells, beta=True):
    """Seeded data of the ARRAYS problem on one level (SURVEY.md §8b ECMG_PROB_ARRAYS; layouts in
    include/ecmg.h): beta_e in [0.5, 2) per element (None if beta is False: beta = 1), f at the 8 Gauss
    points of each element in [-1, 1), g_D per node in [-1, 1), g_R at the 4 Gauss points of every face
    element in [-1, 1)."""
    nx, ny, nz = (int(v) for v in n_cells)
    ne, nn = nx * ny * nz, (nx + 1) * (ny + 1) * (nz + 1)
    u = counter_uniform(seed, ne + 8 * ne + nn + face_gauss_count(n_cells))
    b = 0.5 + 1.5 * u[:ne] if beta else None
    f = 2.0 * u[ne:9 * ne] - 1.0
    g = 2.0 * u[9 * ne:9 * ne + nn] - 1.0
    r = 2.0 * u[9 * ne + nn:] - 1.0
    return b, f, g, r
