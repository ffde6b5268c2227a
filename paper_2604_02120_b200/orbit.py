"""Multi-GPU orbit rendering: the 64-view camera orbit of BASELINE.json
configs[4] partitioned by view across ranks (one process per GPU), finished
frames gathered to rank 0. Views are independent units, so the only exchange
step is the frame gather (no reduction anywhere). Host-side logic only; the
renders run in libgsrender.so."""
from __future__ import annotations


def partition_views(n_views: int, world: int, rank: int) -> range:
    """Contiguous block of views owned by `rank` (equal blocks: world | n_views)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_views % world:
        raise ValueError(f"{n_views} views do not split evenly over {world} ranks")
    per = n_views // world
    return range(rank * per, (rank + 1) * per)


def gather_frames(rgb, T, world: int, rank: int, dist=None):
    """Gathers every rank's [per,3,H,W] / [per,H,W] frames to rank 0.

    Returns (rgb_all [n_views,3,H,W], T_all [n_views,H,W]) on rank 0 (in view
    order, since ranks own contiguous view blocks) and (None, None) elsewhere.
    Uses torch.distributed.gather: NCCL over NVLink on GPUs, gloo on CPU."""
    import torch
    if world == 1:
        return rgb, T
    if dist is None:
        import torch.distributed as dist
    lr = [torch.empty_like(rgb) for _ in range(world)] if rank == 0 else None
    lt = [torch.empty_like(T) for _ in range(world)] if rank == 0 else None
    dist.gather(rgb, lr, dst=0)
    dist.gather(T, lt, dst=0)
    if rank != 0:
        return None, None
    return torch.cat(lr, 0), torch.cat(lt, 0)
