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


def gather_frames_pipelined(rgb, T, world: int, rank: int, group: int, wait_group=None, dist=None, out=None):
    """gather_frames, one view group at a time, overlapped with the rendering.

    rgb [per,3,H,W] / T [per,H,W] are this rank's frames, rendered in view groups of
    `group` by gs_render_views. For each group g, `wait_group(stream, g)` (the C-ABI's
    gs_stream_wait_group) makes a side stream wait until that group has finished
    blending, and an asynchronous NCCL gather of the group's frames is issued on it,
    so the transfer of group g overlaps the rendering of groups g+1, ... The current
    stream waits for every gather before returning. `out`: optional preallocated
    (rgb_all [world,per,3,H,W], T_all [world,per,H,W]) receive buffers on rank 0.
    Returns (rgb_all [world*per,3,H,W], T_all [world*per,H,W]) on rank 0 (view order:
    ranks own contiguous view blocks), (None, None) elsewhere."""
    import contextlib

    import torch
    if world == 1:
        return rgb, T
    if dist is None:
        import torch.distributed as dist
    per = rgb.shape[0]
    if rank == 0:
        if out is None:
            out = (torch.empty((world,) + tuple(rgb.shape), dtype=rgb.dtype, device=rgb.device),
                   torch.empty((world,) + tuple(T.shape), dtype=T.dtype, device=T.device))
        all_rgb, all_T = out
    side = torch.cuda.Stream(device=rgb.device) if rgb.is_cuda else None
    works = []
    for g0 in range(0, per, group):
        sl = slice(g0, min(per, g0 + group))
        if wait_group is not None and side is not None:
            wait_group(side, g0 // group)
        with (torch.cuda.stream(side) if side is not None else contextlib.nullcontext()):
            lr = [all_rgb[r, sl] for r in range(world)] if rank == 0 else None
            lt = [all_T[r, sl] for r in range(world)] if rank == 0 else None
            works.append(dist.gather(rgb[sl], lr, dst=0, async_op=True))
            works.append(dist.gather(T[sl], lt, dst=0, async_op=True))
    for w in works:
        w.wait()
    if side is not None:
        torch.cuda.current_stream(rgb.device).wait_stream(side)
    if rank != 0:
        return None, None
    return all_rgb.view((world * per,) + tuple(rgb.shape[1:])), all_T.view((world * per,) + tuple(T.shape[1:]))
