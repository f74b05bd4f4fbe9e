"""z-slab decomposition on one GPU (virtual slabs: device copies stand in for the NCCL halo
messages, an in-order sum kernel for the allreduce): the sharded Alg. 4 run and
sharded fixed-iteration solves agree with the single-GPU path and with the oracle."""
import numpy as np
import pytest
import torch

import oracle as o
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1506_02983_b200 import Grid, ecmg


def params_for(pid):
    return synth.c5_geometry(0) if pid == o.C5 else None


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("pid,levels,eps,P", [
    (o.C2, 5, 1e-10, 2), (o.C4, 5, 1e-9, 2), (o.C4, 6, 1e-9, 4), (o.C3, 5, 1e-10, 2), (o.C5, 6, 1e-8, 4),
    (o.C2, 6, 1e-10, 8)])
def test_virtual_slab_run(pid, levels, eps, P):
    g1 = Grid(4, levels, pid, params_for(pid))
    u1, ut1 = g1.new_vec(levels - 1), g1.new_vec(levels - 1)
    st1, s1 = g1.run(eps, u1, ut1)
    gp = Grid(4, levels, pid, params_for(pid))
    gp.set_option(ecmg.OPT_VIRTUAL_SLABS, P)
    gp.set_option(ecmg.OPT_SHARD_MIN, 16)   # split the small test levels too
    n_fine = 4 << (levels - 1)
    assert ecmg.slab_partition(n_fine, P, 0)[0]   # the finest level is sharded
    up, utp = gp.new_vec(levels - 1), gp.new_vec(levels - 1)
    stp, sp = gp.run(eps, up, utp)
    assert st1 == 0 and stp == 0
    it1 = [s["iterations"] for s in s1]
    itp = [s["iterations"] for s in sp]
    assert all(abs(a - b) <= 1 for a, b in zip(it1, itp)), (it1, itp)
    assert sp[-1]["rel_res_recur"] <= eps
    a, b = host(up), host(u1)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))
    assert np.max(np.abs(host(utp) - host(ut1))) <= 1e-9 * np.max(np.abs(host(ut1)))
    # and against the oracle
    ost, ostats, ou, out = o.ecmg(4, levels, pid, eps, params=params_for(pid))
    assert np.max(np.abs(a - ou)) <= 1e-9 * np.max(np.abs(ou))


@pytest.mark.parametrize("pid,P", [(o.C2, 2), (o.C3, 2), (o.C5, 4)])
def test_virtual_slab_fixed_iterations(pid, P):
    level = 4   # 64^3: sharded for P = 2 and 4
    n = (64,) * 3
    L = o.Level(n, pid, params=params_for(pid))
    m, _ = L.dirichlet()
    x0 = np.where(~m, synth.random_nodal(14, n), 0.0)
    res = []
    for p in (1, P):
        g = Grid(4, level + 1, pid, params_for(pid))
        if p > 1:
            g.set_option(ecmg.OPT_VIRTUAL_SLABS, p)
            g.set_option(ecmg.OPT_SHARD_MIN, 16)   # split the small test levels too
        u = torch.from_numpy(x0.copy()).cuda()
        st, s = g.solve_level(level, 0.0, 20, u)
        assert st == 0 and s["iterations"] == 20
        res.append(host(u))
    xo, _ = L.jcg(x0, 0.0, 20)
    d_sl = np.max(np.abs(res[1] - res[0])) / np.max(np.abs(res[0]))
    d_or = np.max(np.abs(res[1] - xo)) / np.max(np.abs(xo))
    assert d_sl <= 1e-12 and d_or <= 1e-12, (d_sl, d_or)


def test_nccl_single_rank_selftest():
    # one NCCL rank with every sharded-eligible level forced onto the slab path: exercises dlopen of
    # libnccl, ncclGetUniqueId, ncclCommInitRank and the allreduce -> finalize passes on one GPU
    # (no inter-rank waiting). Run in a subprocess against libecmg_test.so (the -DECMG_TESTING build of the same
    # sources: the force switch is not in the product library); the flag is process-wide.
    import subprocess, sys, os, json
    code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_1506_02983_b200 import Grid, ecmg, PROB
ecmg.LIB_PATH = os.path.join(os.path.dirname(ecmg.LIB_PATH), "libecmg_test.so")   # the -DECMG_TESTING build
nid = ecmg.nccl_unique_id()
g1 = Grid(4, 5, PROB["C2"]); u1 = g1.new_vec(4); st1, s1 = g1.run(1e-10, u1)
d = ecmg.make_dist(0, 1, nid)
gn = Grid(4, 5, PROB["C2"], dist=d); gn.set_option(ecmg.OPT_SHARD_MIN, 16); un = gn.new_vec(4); stn, sn = gn.run(1e-10, un)
gh = Grid(4, 5, PROB["C2"], dist=ecmg.make_dist(0, 1, ecmg.nccl_unique_id())); gh.set_option(ecmg.OPT_SHARD_MIN, 16)
gh.set_option(ecmg.OPT_GRAPH, 0); uh = gh.new_vec(4); sth, sh = gh.run(1e-10, uh)   # the host loop
torch.cuda.synchronize()
a, b, c = un.cpu().numpy(), u1.cpu().numpy(), uh.cpu().numpy()
print(json.dumps(dict(st=[st1, stn, sth], it1=[s["iterations"] for s in s1], itn=[s["iterations"] for s in sn],
                      ith=[s["iterations"] for s in sh], graph_vs_host_bitwise=bool(np.array_equal(a, c)),
                      d=float(np.max(np.abs(a - b)) / np.max(np.abs(b))))))
'''
    env = dict(os.environ, ECMG_TEST_NCCL_SINGLE="1", ECMG_DEBUG="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["st"] == [0, 0, 0]
    assert r["it1"] == r["itn"] == r["ith"]
    assert r["d"] <= 1e-13
    # the sharded levels ran as CUDA graphs with the NCCL allreduce captured inside the WHILE body (a failed
    # capture would fall back to the host loop and say so on stderr under ECMG_DEBUG), bitwise = host loop
    assert "graph capture failed" not in out.stderr, out.stderr[-2000:]
    assert r["graph_vs_host_bitwise"]


@pytest.mark.parametrize("pid,levels,eps,P", [(o.C2, 5, 1e-10, 2), (o.C3, 5, 1e-10, 2), (o.C5, 6, 1e-8, 4),
                                              (o.C4, 6, 1e-9, 8)])
def test_fused_halo_equals_copied_halo(pid, levels, eps, P):
    # ECMG_OPT_FUSED_HALO: the K2 / init passes store their boundary planes straight into the neighbour
    # slabs' halo planes (the kernel code the NCCL ranks run over CUDA-IPC peer memory) instead of a
    # copy after the pass; the halo values are the same, so every iterate is bitwise identical
    res = []
    for fused in (0, 1):
        g = Grid(4, levels, pid, params_for(pid))
        g.set_option(ecmg.OPT_VIRTUAL_SLABS, P)
        g.set_option(ecmg.OPT_SHARD_MIN, 16)   # split the small test levels too
        g.set_option(ecmg.OPT_FUSED_HALO, fused)
        u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
        st, stats = g.run(eps, u, ut)
        assert st == 0
        res.append(([s["iterations"] for s in stats], host(u), host(ut)))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])


@pytest.mark.parametrize("pid,levels,eps,P,fused", [(o.C2, 5, 1e-10, 2, 1), (o.C3, 5, 1e-10, 2, 0),
                                                    (o.C5, 6, 1e-8, 4, 1), (o.C4, 6, 1e-9, 8, 0)])
def test_slab_graph_loop_equals_host_loop(pid, levels, eps, P, fused):
    # ECMG_OPT_GRAPH on sharded levels: one CUDA graph per level (init pass, WHILE node whose body is two
    # iterations of K1 / allreduce / finalize / K2 / allreduce / finalize / halo, true residual), the WHILE
    # condition set by the finalize kernels -- the same kernels in the same order as the host loop, so
    # every iterate is bitwise identical and the counts are equal
    res = []
    for graph in (0, 1):
        g = Grid(4, levels, pid, params_for(pid))
        g.set_option(ecmg.OPT_VIRTUAL_SLABS, P)
        g.set_option(ecmg.OPT_SHARD_MIN, 16)   # split the small test levels too
        g.set_option(ecmg.OPT_FUSED_HALO, fused)
        g.set_option(ecmg.OPT_GRAPH, graph)
        g.set_option(ecmg.OPT_PERS_TMA, 0)   # replicated mid levels: graph vs host loop of the same K1 / K2 too
        u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
        l0 = ecmg.kernel_launches()
        st, stats = g.run(eps, u, ut)
        st2, stats2 = g.run(eps, u, ut)   # second run: the graphs are reused
        assert st == 0 and st2 == 0
        res.append(([s["iterations"] for s in stats], host(u), host(ut), [s["iterations"] for s in stats2],
                    ecmg.kernel_launches() - l0))
    assert res[0][0] == res[1][0] == res[1][3]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
    assert res[1][4] > 0


@pytest.mark.parametrize("pid,levels,eps,P", [(o.C2, 6, 1e-10, 2), (o.C4, 6, 1e-9, 8), (o.C3, 5, 1e-10, 2),
                                              (o.C5, 6, 1e-8, 4)])
def test_hybrid_cascade_vs_slab_loop(pid, levels, eps, P):
    # ECMG_OPT_SLAB_HYBRID: the replicated levels (before the first sharded one) run through the single-GPU
    # path (one-CTA / persistent / graph solves, setup ahead), then their last two solutions seed the slab
    # driver; the slab driver's host loop for every level is the reference: counts +-1, solutions within
    # rounding, and the per-level statistics of every level are filled
    res = []
    for hyb in (1, 0):
        g = Grid(4, levels, pid, params_for(pid))
        g.set_option(ecmg.OPT_VIRTUAL_SLABS, P)
        g.set_option(ecmg.OPT_SHARD_MIN, 16)   # split the small test levels too
        g.set_option(ecmg.OPT_SLAB_HYBRID, hyb)
        u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
        st, stats = g.run(eps, u, ut)
        assert st == 0
        assert all(s["iterations"] > 0 and s["rel_res_true"] > 0 for s in stats)
        res.append(([s["iterations"] for s in stats], host(u), host(ut)))
    assert all(abs(a - b) <= 1 for a, b in zip(res[0][0], res[1][0])), (res[0][0], res[1][0])
    for k in (1, 2):
        assert np.max(np.abs(res[0][k] - res[1][k])) <= 1e-9 * np.max(np.abs(res[1][k]))


@pytest.mark.parametrize("pid,levels,eps,P", [(o.C2, 6, 1e-10, 2), (o.C5, 6, 1e-8, 4), (o.C3, 5, 1e-10, 2)])
def test_slab_finest_setup_ahead_bitwise(pid, levels, eps, P):
    # in the hybrid cascade the finest (split) level's setup runs ahead on the slab driver's stream while
    # the replicated levels are solved (own b / beta buffers); same kernels on the same data as the in-line
    # setup, so every iterate is bitwise equal; the second run on the same grid sets up ahead again
    res = []
    for ahead in (0, 1):
        g = Grid(4, levels, pid, params_for(pid))
        g.set_option(ecmg.OPT_VIRTUAL_SLABS, P)
        g.set_option(ecmg.OPT_SHARD_MIN, 16)
        g.set_option(ecmg.OPT_SETUP_AHEAD, ahead)
        u, ut = g.new_vec(levels - 1), g.new_vec(levels - 1)
        for _ in range(2):
            st, stats = g.run(eps, u, ut)
            assert st == 0
        res.append(([s["iterations"] for s in stats], host(u), host(ut)))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
