"""The oracle's threaded mode (orc_set_threads) is the serial program run faster, not a second program:
every assembled entry, load, lifted right-hand side, A_ff p, JCG iterate, EXP_finite / EXP_true value and
Alg. 4 statistic is BITWISE equal to the single-threaded oracle's (row loops in parallel, element
contributions to a row in the same lexicographic order, every reduction serial in node order). The
full-size goldens (tests/golden/fullsize_*.json) are written in this mode, so this test is what lets them
stand for the serial oracle."""
import numpy as np
import pytest

import oracle as o
import synth

CASES = [(o.C1, (16, 16, 16), None), (o.C3, (16, 16, 16), None), (o.C4, (16, 16, 16), None),
         (o.C5, (16, 16, 16), "c5"), (o.P1, (12, 8, 16), None), (o.P2, (10, 4, 5), None),
         (o.PATCH_ROBIN_XY, (8, 12, 8), None)]


def _params(tag):
    return synth.c5_geometry(0) if tag == "c5" else None


@pytest.fixture
def threads4():
    prev = o.set_threads(4)
    yield
    o.set_threads(prev)


def _level_dump(n, pid, params):
    L = o.Level(n, pid, params=params)
    b, nb = L.rhs()
    m, g = L.dirichlet()
    p = synth.random_nodal(11, n)
    x0 = synth.random_nodal(14, n)
    x, st = L.jcg(np.where(m, 0.0, x0), 0.0, 7)   # 7 fixed iterations
    w = L.exp_finite(synth.random_nodal(13, tuple(c // 2 for c in n)), synth.random_nodal(12, tuple(c // 4 for c in n))) \
        if all(c % 4 == 0 for c in n) else None
    t = L.exp_true(p, synth.random_nodal(13, tuple(c // 2 for c in n))) if all(c % 2 == 0 for c in n) else None
    return [L.matrix(), L.load(), b, np.array([nb]), m, g, L.apply(p), x, np.array([st["rel_recur"], st["rel_true"]]),
            w, t]


@pytest.mark.parametrize("pid,n,tag", CASES)
def test_threaded_level_bitwise(pid, n, tag, threads4):
    got = _level_dump(n, pid, _params(tag))
    o.set_threads(1)
    ref = _level_dump(n, pid, _params(tag))
    for a, b in zip(got, ref):
        if a is None:
            assert b is None
            continue
        assert np.array_equal(a, b)


@pytest.mark.parametrize("pid,levels,eps,tag", [(o.C1, 4, 1e-8, None), (o.C3, 4, 1e-10, None), (o.C5, 4, 1e-8, "c5"),
                                                 (o.P2, 3, 1e-9, None)])
def test_threaded_ecmg_bitwise(pid, levels, eps, tag, threads4):
    n0 = (10, 4, 5) if pid == o.P2 else 4
    res_t = o.ecmg(n0, levels, pid, eps, params=_params(tag), want_w=True)
    o.set_threads(1)
    res_1 = o.ecmg(n0, levels, pid, eps, params=_params(tag), want_w=True)
    assert res_t[0] == res_1[0] == 0
    keep = [c for c in range(o.NSTAT) if not o.STAT_FIELDS[c].startswith("t_")]   # wall times differ
    assert np.array_equal(res_t[1][:, keep], res_1[1][:, keep], equal_nan=True)
    for a, b in zip(res_t[2:], res_1[2:]):
        assert np.array_equal(a, b)


def test_threaded_arrays_bitwise(threads4):
    n = (12, 8, 16)
    faces = [0, 1, 1, 0, 1, 0]
    alpha = [0.0, 0.5, 2.0, 0.0, 1.5, 0.0]
    arr = synth.random_problem_arrays(21, n)
    A = o.Level.from_arrays(n, faces, alpha, *arr)
    got = [A.matrix(), A.load(), A.rhs()[0]]
    o.set_threads(1)
    B = o.Level.from_arrays(n, faces, alpha, *arr)
    for a, b in zip(got, [B.matrix(), B.load(), B.rhs()[0]]):
        assert np.array_equal(a, b)


def test_set_threads_rejects_zero():
    with pytest.raises(ValueError):
        o.set_threads(0)
    assert o.max_threads() >= 1
