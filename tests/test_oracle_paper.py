"""The oracle reproduces the numbers the paper prints (Tables 1, 6-10) -- values typed from
PAPER.md into tests/golden/paper_tables.json, each block with its citation -- and the error
orders the paper's analysis fixes.

Reading recorded in DESIGN.md ("R-EXP"): the paper's printed ||W-U||, r_h, RRe and iteration
counts are reproduced by Remark 2's 27-node Lagrange EXP_finite, not by the 20-node
Serendipity variant the text says it reports. FE-solution quantities (||U-u||, ||u~-u||)
do not depend on the variant and match under both."""
import json
import os

import numpy as np
import pytest

import oracle as o

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
S = {n: i for i, n in enumerate(o.STAT_FIELDS)}


def rel(a, b):
    return abs(a - b) / abs(b)


@pytest.fixture(scope="module")
def p1_1e9():
    # Problem 1, coarsest 8^3, levels 8,16,32,64; eps = 1e-9
    out = {}
    for var in (0, 1):
        st, stats, u, ut = o.ecmg(8, 4, o.P1, 1e-9, exp_variant=var)
        assert st == 0
        out[var] = stats
    return out


def test_p1_table6_7_lagrange(p1_1e9):
    g = GOLD["p1_eps1e-9"]
    st = p1_1e9[1]
    for lev, k in ((2, 0), (3, 1)):   # 32^3, 64^3
        row = st[lev]
        assert int(row[S["iterations"]]) == g["iters"][k]
        assert rel(row[S["rel_true"]], g["rre"][k]) < 0.02
        for key in ("err_l2", "err_linf", "err_tilde_l2", "err_tilde_linf", "err_w_l2", "err_w_linf", "r_h"):
            assert rel(row[S[key]], g[key][k]) < 0.01, (key, k, row[S[key]], g[key][k])


def test_p1_serendipity_orders(p1_1e9):
    g = GOLD["p1_eps1e-9"]
    st = p1_1e9[0]
    for lev, k in ((2, 0), (3, 1)):
        row = st[lev]
        # FE-solution quantities are variant independent and match the paper
        for key in ("err_l2", "err_linf", "err_tilde_l2", "err_tilde_linf"):
            assert rel(row[S[key]], g[key][k]) < 0.01
        assert row[S["rel_recur"]] <= 1e-9
    # third-order guess and r_h halving per level
    order_w = np.log2(st[2, S["err_w_l2"]] / st[3, S["err_w_l2"]])
    assert abs(order_w - 3.0) < 0.15
    assert abs(st[2, S["r_h"]] / st[3, S["r_h"]] - 2.0) < 0.2
    assert abs(np.log2(st[2, S["err_linf"]] / st[3, S["err_linf"]]) - 2.0) < 0.05
    assert abs(np.log2(st[2, S["err_tilde_linf"]] / st[3, S["err_tilde_linf"]]) - 4.0) < 0.1


def test_p1_table1_iterations_jcg_cg():
    g = GOLD["p1_eps1e-8"]
    st, sj, _, _ = o.ecmg(8, 4, o.P1, 1e-8, exp_variant=1, precond=True)
    st2, sc, _, _ = o.ecmg(8, 4, o.P1, 1e-8, exp_variant=1, precond=False)
    assert [int(v) for v in sj[2:, S["iterations"]]] == g["iters_jcg"][:2]
    assert [int(v) for v in sc[2:, S["iterations"]]] == g["iters_cg"][:2]
    assert rel(sj[2, S["rel_true"]], g["rre"][0]) < 0.01
    assert rel(sj[3, S["rel_true"]], g["rre"][1]) < 0.01


@pytest.mark.slow
def test_p1_table1_128():
    g = GOLD["p1_eps1e-8"]
    _, sj, _, _ = o.ecmg(8, 5, o.P1, 1e-8, exp_variant=1, precond=True)
    _, sc, _, _ = o.ecmg(8, 5, o.P1, 1e-8, exp_variant=1, precond=False)
    assert [int(v) for v in sj[2:, S["iterations"]]] == g["iters_jcg"]
    assert [int(v) for v in sc[2:, S["iterations"]]] == g["iters_cg"]


def test_p2_tables8_9():
    g = GOLD["p2_eps1e-12"]
    st, stats, _, _ = o.ecmg((10, 4, 5), 4, o.P2, 1e-12, exp_variant=1)
    assert st == 0
    for lev, k in ((2, 0), (3, 1)):
        row = stats[lev]
        for key in ("err_l2", "err_linf", "err_tilde_l2", "err_tilde_linf"):
            assert rel(row[S[key]], g[key][k]) < 0.01, (key, k)
        for key in ("err_w_l2", "err_w_linf", "r_h"):
            assert rel(row[S[key]], g[key][k]) < 0.10, (key, k)
        assert abs(row[S["iterations"]] - g["iters"][k]) <= 0.25 * g["iters"][k]   # bands


def test_p3_table10():
    g = GOLD["p3_eps1e-11"]
    st, stats, _, _ = o.ecmg(8, 4, o.P3, 1e-11, exp_variant=1)
    assert st == 0
    for lev, k in ((2, 0), (3, 1)):
        row = stats[lev]
        for key in ("err_l2", "err_tilde_l2", "err_w_l2", "r_h"):
            assert rel(row[S[key]], g[key][k]) < 0.03, (key, k)
    # singular solution: extrapolated order ~3, not 4
    assert abs(np.log2(stats[2, S["err_tilde_l2"]] / stats[3, S["err_tilde_l2"]]) - 2.97) < 0.1


@pytest.mark.parametrize("pid,tilde_order", [(o.C1, 4.0), (o.C2, 4.0), (o.C3, 4.0), (o.C4, 3.0)])
def test_configs_orders(pid, tilde_order):
    # C1-C4 at tight eps: FE order 2, extrapolated order 4 (3 for the r^{3/2} singularity),
    # third-order guess
    st, stats, _, _ = o.ecmg(4, 5, pid, 1e-12)
    assert st == 0
    a, b = stats[3], stats[4]   # 32^3 -> 64^3
    assert abs(np.log2(a[S["err_l2"]] / b[S["err_l2"]]) - 2.0) < 0.06
    assert abs(np.log2(a[S["err_tilde_l2"]] / b[S["err_tilde_l2"]]) - tilde_order) < 0.25
    assert abs(np.log2(a[S["err_w_l2"]] / b[S["err_w_l2"]]) - 3.0) < 0.3
