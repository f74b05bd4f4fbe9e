"""The oracle's one-row-at-a-time evaluations (used for parity at full size, where the assembled level
does not fit in host memory) against the assembled level, bitwise: every row is the same sum of the same
element / face matrix entries in the same order, and the EXP node bodies are the bulk loops' bodies."""
import numpy as np
import pytest

import oracle as o
import synth


def params_for(pid):
    if pid == o.C5:
        return synth.c5_geometry(0)
    if pid == o.PATCH_LAYERED:
        return synth.layered_only(0)
    return None


CASES = [(o.C1, (8, 8, 8)), (o.C3, (8, 8, 8)), (o.C4, (8, 8, 8)), (o.C5, (16, 16, 16)), (o.P1, (8, 8, 8)),
         (o.P2, (10, 4, 5)), (o.PATCH_ROBIN_XY, (8, 8, 8)), (o.PATCH_LAYERED, (8, 8, 8))]


def all_nodes(n):
    iz, iy, ix = np.meshgrid(np.arange(n[2] + 1), np.arange(n[1] + 1), np.arange(n[0] + 1), indexing="ij")
    return np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)


@pytest.mark.parametrize("pid,n", CASES)
def test_rows_equal_assembled_level(pid, n):
    L = o.Level(n, pid, params=params_for(pid))
    p = synth.random_nodal(11, n)
    q, b = o.rows(n, pid, all_nodes(n), p, params=params_for(pid))
    assert np.array_equal(q, L.apply(p))     # (A_ff p)_i, Dirichlet rows 0
    assert np.array_equal(b, L.rhs()[0])     # lifted right-hand side b_f


@pytest.mark.parametrize("pid,n", [(o.C1, (16, 16, 16)), (o.C3, (16, 16, 16)), (o.P2, (40, 16, 20)),
                                   (o.P1, (16, 16, 16))])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_exp_nodes_equal_bulk(pid, n, which):
    L = o.Level(n, pid, params=params_for(pid))
    nodes = all_nodes(n)
    if which < 2:
        a = synth.random_nodal(13, tuple(c // 2 for c in n))
        c = synth.random_nodal(12, tuple(c // 4 for c in n))
        ref = L.exp_finite(a, c, which)
    else:
        a = synth.random_nodal(11, n)
        c = synth.random_nodal(13, tuple(v // 2 for v in n))
        ref = L.exp_true(a, c)
    got = o.exp_nodes(n, pid, which, a, c, nodes, params=params_for(pid))
    assert np.array_equal(got, ref)


def test_rows_reject_bad_nodes():
    with pytest.raises(ValueError):
        o.rows((8, 8, 8), o.C1, [[9, 0, 0]])
    with pytest.raises(ValueError):
        o.exp_nodes((6, 8, 8), o.C1, 0, np.zeros(4 * 5 * 5), np.zeros(8), [[0, 0, 0]])


@pytest.mark.parametrize("pid,n", [(o.C3, (8, 8, 8)), (o.P2, (10, 4, 5))])
def test_rows_diagonal(pid, n):
    # the Jacobi diagonal A_ii: (A e_i)_i of the assembled level for a few separated free nodes
    L = o.Level(n, pid, params=params_for(pid))
    m, _ = L.dirichlet()
    nodes = all_nodes(n)
    free = np.nonzero(~m)[0][::37]
    _, _, dg = o.rows(n, pid, nodes[free], params=params_for(pid), diag=True)
    for k, i in enumerate(free):
        e = np.zeros(L.N)
        e[i] = 1.0
        assert dg[k] == L.apply(e)[i]
