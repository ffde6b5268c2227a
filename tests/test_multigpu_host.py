"""N > 1 host path on CPU: view partition and the frame gather (gloo, world size 2)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_02120_b200.orbit import (band_pixel_rows, gather_bands, gather_frames, gather_frames_pipelined,
                                         gather_plan, partition_views)


def test_partition_covers_views_once():
    for world in (1, 2, 4, 8):
        seen = [v for r in range(world) for v in partition_views(64, world, r)]
        assert seen == list(range(64))
    with pytest.raises(ValueError):
        partition_views(64, 3, 0)


def test_gather_plan():
    """One preprocess launch per rank and step while the block fits a view group (16),
    gather chunks of a quarter block: N = 1, 2, 4, 8 ranks of the 64-view orbit."""
    assert [gather_plan(64 // n) for n in (1, 2, 4, 8)] == [(16, 16), (16, 8), (16, 4), (8, 2)]
    assert gather_plan(1) == (1, 1) and gather_plan(3) == (3, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = partition_views(8, world, rank)
    H, W = 3, 5
    # frame content encodes its view id, as a render of view v would
    rgb = torch.stack([torch.full((3, H, W), float(v)) for v in views])
    T = torch.stack([torch.full((H, W), -float(v)) for v in views])
    # tile-row split of one 70-row view (5 tile rows, bands of 2 and 3 tile rows): each
    # rank fills only its band; the rest is garbage that must not leak into the result
    Hv, Wv = 70, 9
    frgb = torch.full((3, Hv, Wv), -7.0)
    fT = torch.full((Hv, Wv), -7.0)
    yy = torch.arange(Hv, dtype=torch.float32).view(Hv, 1).expand(Hv, Wv)
    r = band_pixel_rows(Hv, rank, world)
    frgb[:, r.start:r.stop] = yy[r.start:r.stop]
    fT[r.start:r.stop] = -yy[r.start:r.stop]
    brgb, bT = gather_bands(frgb, fT, world, rank)
    if rank == 0:
        assert torch.equal(brgb, yy.expand(3, Hv, Wv)) and torch.equal(bT, -yy)
    a, b = gather_frames(rgb, T, world, rank)
    # the chunk-pipelined gather (chunks of 3 views: a ragged last chunk)
    c, d = gather_frames_pipelined(rgb, T, world, rank, 3)
    if rank == 0:
        assert torch.equal(a, c) and torch.equal(b, d)
        q.put((a.clone(), b.clone()))
    else:
        assert c is None and d is None
    dist.barrier()
    dist.destroy_process_group()


def test_gather_frames_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    rgb, T = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert rgb.shape == (8, 3, 3, 5) and T.shape == (8, 3, 5)
    for v in range(8):
        assert (rgb[v] == v).all() and (T[v] == -v).all()


def test_band_rows_partition_the_frame():
    for H in (1, 16, 45, 1080, 8400):
        for n in (1, 2, 3, 5, 8):
            rows = [v for b in range(n) for v in band_pixel_rows(H, b, n)]
            assert rows == list(range(H))
