"""Independent pin of the oracle's C5 data (BASELINE.json configs[4]; Eq. (bvp)): the element beta
(layers + boxes, SURVEY.md §8d "C5 recipe": beta_e = the value of the LAST box containing the element
centroid, else the layer containing its z, strict z < z_l) and the Gaussian source f at the 2x2x2 Gauss
points are sampled here in numpy straight from the committed fixture tests/golden/c5_seed0.json, and handed
to the oracle's ARRAYS problem (caller data, itself pinned in test_oracle_arrays.py). The registry C5 level
must be the same level: a wrong box test (<= vs <, an axis mix-up, first box winning instead of the last),
a wrong layer index, or a wrong source formula (sigma^2 vs 2 sigma^2, a shifted centre) changes beta or f
on whole element sets and fails it."""
import json
import os

import numpy as np
import pytest

import oracle as o
import synth
from arrays_data import element_points

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c5_seed0.json")))


def c5_beta_numpy(cx, cy, cz):
    z_l = np.array(FIX["heights"])
    layer = np.searchsorted(z_l, cz, side="right")   # first l with z < z_l (strict), else 7
    beta = np.array(FIX["layer_beta"])[layer]
    for (bx, by, bz, sx, sy, sz, bv) in FIX["boxes"]:   # in draw order: a later box overrides
        inside = (np.abs(cx - bx) < sx) & (np.abs(cy - by) < sy) & (np.abs(cz - bz) < sz)
        beta = np.where(inside, bv, beta)
    return beta


def c5_f_numpy(x, y, z):
    x0, s, amp = FIX["x0"], FIX["sigma"], FIX["amplitude"]
    d2 = (x - x0[0]) ** 2 + (y - x0[1]) ** 2 + (z - x0[2]) ** 2
    return amp * np.exp(-d2 / (2.0 * s * s))


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("n", [(32, 32, 32), (40, 24, 36)])
def test_c5_registry_equals_numpy_sampling(n):
    lo, hi = (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    (cx, cy, cz), (X, Y, Z) = element_points(n, lo, hi)
    beta = c5_beta_numpy(cx, cy, cz)
    # the sample is discriminating: every layer and every box owns elements at this resolution
    z_l = np.array(FIX["heights"])
    assert len(np.unique(np.searchsorted(z_l, cz, side="right"))) == 8
    for (bx, by, bz, sx, sy, sz, bv) in FIX["boxes"]:
        assert np.any((np.abs(cx - bx) < sx) & (np.abs(cy - by) < sy) & (np.abs(cz - bz) < sz) & (beta == bv))
    f = c5_f_numpy(X, Y, Z)
    faces = [o.DIRICHLET] * 6
    arr = o.Level.from_arrays(n, faces, [0.0] * 6, beta_e=beta.reshape(-1), f_q=f.reshape(-1), gD=None, gR=None)
    reg = o.Level(n, o.C5, params=synth.c5_geometry(0))
    assert np.array_equal(arr.matrix(), reg.matrix())          # same beta_e on every element: bitwise
    assert rel(arr.load(), reg.load()) <= 1e-13                 # exp: numpy vs glibc, a few ulp
    (ba, na), (br, nr) = arr.rhs(), reg.rhs()
    assert rel(ba, br) <= 1e-13 and abs(na - nr) <= 1e-13 * nr
    m, g = reg.dirichlet()
    assert np.all(g == 0.0) and int(m.sum()) == (n[0] + 1) * (n[1] + 1) * (n[2] + 1) - (n[0] - 1) * (n[1] - 1) * (n[2] - 1)


def test_c5_numpy_sampler_is_not_trivial():
    # the readings a plausible bug would take give a DIFFERENT beta / f (so the test above can fail). The
    # four seed-0 boxes do not overlap on element centroids, so "last box wins" is not separable here.
    n = (32, 32, 32)
    (cx, cy, cz), (X, Y, Z) = element_points(n, (0, 0, 0), (1, 1, 1))
    beta = c5_beta_numpy(cx, cy, cz)
    z_l = np.array(FIX["heights"])
    layers_only = np.array(FIX["layer_beta"])[np.searchsorted(z_l, cz, side="right")]
    assert not np.array_equal(beta, layers_only)                   # boxes dropped
    swapped = layers_only.copy()
    for (bx, by, bz, sx, sy, sz, bv) in FIX["boxes"]:               # x / y axes of the box test mixed up
        inside = (np.abs(cy - bx) < sx) & (np.abs(cx - by) < sy) & (np.abs(cz - bz) < sz)
        swapped = np.where(inside, bv, swapped)
    assert not np.array_equal(beta, swapped)
    off_by_one = np.array(FIX["layer_beta"])[np.minimum(np.searchsorted(z_l, cz, side="left") + 1, 7)]
    assert not np.array_equal(layers_only, off_by_one)             # wrong layer index
    f = c5_f_numpy(X, Y, Z)
    x0, s = FIX["x0"], FIX["sigma"]
    f_wrong = np.exp(-((X - x0[0]) ** 2 + (Y - x0[1]) ** 2 + (Z - x0[2]) ** 2) / (s * s))
    assert rel(f_wrong, f) > 0.1
