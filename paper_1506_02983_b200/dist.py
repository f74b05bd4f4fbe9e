"""torch.distributed plumbing for the z-slab path (argument marshalling only): rank 0 creates the
128-byte NCCL unique id, every rank receives it by broadcast, and the ecmg_dist struct is built."""
from __future__ import annotations

from . import ecmg


def broadcast_nccl_id(make_id=None, device=None) -> bytes:
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    raw = (make_id or ecmg.nccl_unique_id)() if rank == 0 else bytes(128)
    t = torch.tensor(list(raw), dtype=torch.uint8, device=device or "cpu")
    dist.broadcast(t, src=0)
    return bytes(t.cpu().tolist())


def ecmg_dist_from_torch(make_id=None, device=None):
    import torch.distributed as dist
    nid = broadcast_nccl_id(make_id, device)
    return ecmg.make_dist(dist.get_rank(), dist.get_world_size(), nid)
