"""Fused frame gather (SURVEY 8(e) fused variant) on one GPU: two processes, rank 1
maps rank 0's frame buffers through CUDA IPC and renders its views straight into them
(on a multi-GPU box the same mapping is peer memory over NVLink). Frames must equal a
single-process render of all views."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_02120_b200 import Context, camera, opts, scene_to_device, synth
        from paper_2604_02120_b200.orbit import partition_views, share_frames
        torch.cuda.set_device(0)
        scene = synth.unbounded_scene(30000, 113, sh_degree=3)
        cams = synth.orbit_cameras(8, 160, 112, 1.0)
        o = opts((0.1, 0.2, 0.3), sh_degree=3, flags=16)
        own_rgb = torch.full((8, 3, 112, 160), float("nan"), device="cuda") if rank == 0 else None
        own_T = torch.full((8, 112, 160), float("nan"), device="cuda") if rank == 0 else None
        rgb_all, T_all = share_frames(own_rgb, own_T, rank, dist)
        mine = partition_views(8, world, rank)
        ctx = Context(0, max_points=scene.n, max_keys=1 << 22, max_w=160, max_h=112)
        ctx.gs_set_view_group(2, True)
        st = scene_to_device(scene)
        ctx.gs_render_views(st, [camera(cams[v]) for v in mine], 160, 112, o,
                            rgb_all[mine.start:mine.stop], T_all[mine.start:mine.stop])
        torch.cuda.synchronize()
        dist.barrier()   # every rank's writes into rank 0's buffers are complete
        if rank == 0:
            ref_rgb = torch.empty_like(rgb_all)
            ref_T = torch.empty_like(T_all)
            ctx.gs_render_views(st, [camera(c) for c in cams], 160, 112, o, ref_rgb, ref_T)
            torch.cuda.synchronize()
            q.put((bool(torch.equal(rgb_all, ref_rgb)), bool(torch.equal(T_all, ref_T)),
                   bool(torch.isnan(rgb_all).any())))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_fused_frame_gather_through_ipc_two_processes():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    eq_rgb, eq_T, has_nan = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert eq_rgb and eq_T and not has_nan
