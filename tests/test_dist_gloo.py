"""Host logic of the z-slab path with torch.distributed on CPU (gloo, world size 2): the partition
computed independently on every rank tiles each level exactly once and nests across levels, and
the NCCL unique id reaches every rank unchanged. No GPU."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import __graft_entry__ as ge


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1506_02983_b200 import dist as edist
        from paper_1506_02983_b200 import ecmg
        # partition on every level of C4 (4^3 -> 512^3) and C5 (-> 1024^3), for P = world and 8
        out = {}
        for P in (world, 4, 8):
            for n in (4, 8, 16, 32, 64, 128, 256, 512, 1024):
                if rank < P:
                    out[(P, n)] = ecmg.slab_partition(n, P, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        # NCCL id plumbing (a fixed test id: the real one needs libnccl / a GPU box)
        nid = edist.broadcast_nccl_id(make_id=lambda: bytes(range(128)))
        d = ecmg.make_dist(dist.get_rank(), dist.get_world_size(), nid)
        results[rank] = dict(parts=gathered, nid=nid, drank=d.rank, dn=d.nranks, did=bytes(d.nccl_id))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_results():
    ge.build_lib()
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    return dict(results)


def test_nccl_id_broadcast(gloo_results):
    ids = [gloo_results[r]["nid"] for r in range(2)]
    assert ids[0] == ids[1] == bytes(range(128))
    for r in range(2):
        assert gloo_results[r]["drank"] == r and gloo_results[r]["dn"] == 2
        assert gloo_results[r]["did"] == bytes(range(128))


def test_partition_tiles_and_nests(gloo_results):
    parts = gloo_results[0]["parts"]          # every rank's view, gathered
    assert parts == gloo_results[1]["parts"]
    from paper_1506_02983_b200 import ecmg
    for P in (2, 4, 8):
        prev = None
        for n in (4, 8, 16, 32, 64, 128, 256, 512, 1024):
            views = [ecmg.slab_partition(n, P, r) for r in range(P)]
            if P == 2:   # what the two gloo ranks computed on their own
                assert [parts[r][(2, n)] for r in range(2)] == views
            sharded = views[0][0]
            assert all(v[0] == sharded for v in views)
            if not sharded:
                assert all(v[1:] == (0, n + 1) for v in views)
                assert not (n % (4 * P) == 0 and n // P >= 16)
                continue
            # the owned planes tile [0, n] exactly once; slab boundaries are multiples of 4
            covered = []
            for r, (_, lo, hi) in enumerate(views):
                assert lo % 4 == 0 and (hi % 4 == 0 or hi == n + 1)
                assert hi - lo >= 16
                covered += list(range(lo, hi))
            assert covered == list(range(n + 1))
            # nesting: a sharded level's slab boundaries halve onto the coarser level's boundaries
            if prev is not None and prev[0]:
                for r in range(P):
                    assert views[r][1] == 2 * prev[1][r]
            prev = (True, [v[1] for v in views])


def test_partition_rejects_bad_args():
    ge.build_lib()
    from paper_1506_02983_b200 import ecmg
    with pytest.raises(ecmg.EcmgError):
        ecmg.slab_partition(64, 2, 2)
    with pytest.raises(ecmg.EcmgError):
        ecmg.slab_partition(0, 1, 0)
