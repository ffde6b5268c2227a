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


def gather_frames_pipelined(rgb, T, world: int, rank: int, chunk: int, wait_views=None, dist=None, out=None):
    """gather_frames, a chunk of views at a time, overlapped with the rendering.

    rgb [per,3,H,W] / T [per,H,W] are this rank's frames, rendered in view order by
    gs_render_views. For each chunk [v0, v1) of `chunk` views, `wait_views(stream, v1 - 1)`
    (the C-ABI's gs_stream_wait_view) makes a side stream wait until those views have
    finished blending, and an asynchronous NCCL gather of the chunk's frames is issued on
    it, so the transfer of chunk k overlaps the rendering of the later views; the chunk is
    independent of the view group the scene is read in. The current stream waits for every
    gather before returning. `out`: optional preallocated (rgb_all [world,per,3,H,W],
    T_all [world,per,H,W]) receive buffers on rank 0. Returns (rgb_all [world*per,3,H,W],
    T_all [world*per,H,W]) on rank 0 (view order: ranks own contiguous view blocks),
    (None, None) elsewhere."""
    import contextlib

    import torch
    if world == 1:
        return rgb, T
    if dist is None:
        import torch.distributed as dist
    per = rgb.shape[0]
    chunk = max(1, int(chunk))
    if rank == 0:
        if out is None:
            out = (torch.empty((world,) + tuple(rgb.shape), dtype=rgb.dtype, device=rgb.device),
                   torch.empty((world,) + tuple(T.shape), dtype=T.dtype, device=T.device))
        all_rgb, all_T = out
    side = torch.cuda.Stream(device=rgb.device) if rgb.is_cuda else None
    works = []
    for v0 in range(0, per, chunk):
        sl = slice(v0, min(per, v0 + chunk))
        if wait_views is not None and side is not None:
            wait_views(side, sl.stop - 1)
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


def gather_plan(per: int, max_group: int = 16):
    """(view group, gather chunk) for a rank that renders `per` views: the whole block in
    one preprocess launch when it fits a view group (the scene is read once per rank and
    step), the gather in chunks of a quarter of the block (at least 1 view), so that only
    the last chunk's transfer trails the rendering."""
    group = max(1, min(max_group, per))
    return group, max(1, per // 4)


def band_pixel_rows(H: int, band: int, n_bands: int) -> range:
    """Pixel rows of row band `band` of `n_bands` (the C-ABI's gs_opts.band / n_bands:
    tile rows [band*gy/n, (band+1)*gy/n), gy = ceil(H/16))."""
    gy = (H + 15) // 16
    if n_bands <= 1:
        return range(0, H)
    y0, y1 = band * gy // n_bands, (band + 1) * gy // n_bands
    return range(16 * y0, min(H, 16 * y1))


def gather_bands(rgb, T, n_bands: int, rank: int, dist=None):
    """Tile-row split of ONE view across ranks (SURVEY 8(e) option): rank r rendered
    band r of `n_bands` (= world size) into its full-size rgb [3,H,W] / T [H,W] (other
    rows unwritten). Gathers the bands to rank 0 (NCCL over NVLink on GPUs, gloo on
    CPU; bands padded to the tallest one) and returns the assembled (rgb, T) there,
    (None, None) elsewhere. No reduction: every pixel comes from exactly one rank."""
    import torch
    if n_bands == 1:
        return rgb, T
    if dist is None:
        import torch.distributed as dist
    H, W = T.shape
    rows = [band_pixel_rows(H, b, n_bands) for b in range(n_bands)]
    hmax = max(len(r) for r in rows)
    mine = rows[rank]
    prgb = torch.zeros((3, hmax, W), dtype=rgb.dtype, device=rgb.device)
    pT = torch.zeros((hmax, W), dtype=T.dtype, device=T.device)
    prgb[:, :len(mine)] = rgb[:, mine.start:mine.stop]
    pT[:len(mine)] = T[mine.start:mine.stop]
    lr = [torch.empty_like(prgb) for _ in range(n_bands)] if rank == 0 else None
    lt = [torch.empty_like(pT) for _ in range(n_bands)] if rank == 0 else None
    dist.gather(prgb, lr, dst=0)
    dist.gather(pT, lt, dst=0)
    if rank != 0:
        return None, None
    out_rgb = torch.empty_like(rgb)
    out_T = torch.empty_like(T)
    for b, r in enumerate(rows):
        out_rgb[:, r.start:r.stop] = lr[b][:, :len(r)]
        out_T[r.start:r.stop] = lt[b][:len(r)]
    return out_rgb, out_T


def share_frames(frames_rgb, frames_T, rank: int, dist=None):
    """Fused frame "gather" (SURVEY 8(e) fused variant): rank 0 owns the orbit's frame
    buffers [n_views,3,H,W] / [n_views,H,W]; every other rank maps them through CUDA IPC
    (peer memory over NVLink, peer access enabled lazily by the mapping) and its blend
    writes its views' pixels straight into rank 0's buffers -- no separate collective
    and no extra copy. Pass frames_rgb / frames_T on rank 0 (None elsewhere); returns the
    tensors every rank renders into (on rank r, views of rank 0's memory). The handles are
    exchanged with broadcast_object_list (gloo or NCCL); the caller keeps rank 0's
    buffers alive and orders the writes against rank 0's reads with a barrier."""
    from torch.multiprocessing.reductions import reduce_tensor
    if dist is None:
        import torch.distributed as dist
    payload = [None, None]
    if rank == 0:
        payload = [reduce_tensor(frames_rgb)[1], reduce_tensor(frames_T)[1]]
    dist.broadcast_object_list(payload, src=0)
    if rank == 0:
        return frames_rgb, frames_T
    from torch.multiprocessing.reductions import rebuild_cuda_tensor
    return rebuild_cuda_tensor(*payload[0]), rebuild_cuda_tensor(*payload[1])
