"""Debug: is the async host entry point's completion signalled on the caller's stream after
the bench's other sections ran? Times K async calls with events and with the wall clock,
before and after a row-band render, an intersection-mode orbit and an A/B orbit."""
import os, sys, time, math
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2604_02120_b200 import (Context, camera, opts, scene_to_device, scene_to_host, synth, GS_BLEND_TC,
                                   GS_BLEND_DIRECT, GS_FLAG_OBOX, GS_FLAG_TIMING, GS_FLAG_TIGHT)
scene, cams, bg = synth.make_config("C5", views=64)
W, H = cams[0].W, cams[0].H
my = [camera(c) for c in cams]
ctx = Context(0, max_points=scene.n, max_keys=48 << 20, max_w=W, max_h=H)
ctx.gs_set_view_group(16, True)
st = scene_to_device(scene)
stream = torch.cuda.current_stream()
hs = scene_to_host(scene, pinned=True)
h_rgb = torch.empty((64, 3, H, W), pin_memory=True)
h_T = torch.empty((64, H, W), pin_memory=True)
o = opts(bg, sh_degree=scene.sh_degree, flags=GS_FLAG_OBOX)
out_rgb = torch.empty((64, 3, H, W), device="cuda")
out_T = torch.empty((64, H, W), device="cuda")

def e2e(tag, K=6):
    for _ in range(2):
        ctx.gs_render_views_host(hs, my, W, H, o, h_rgb, h_T, stream, async_=True)
    torch.cuda.synchronize()
    ctx.gs_render_views_host(hs, my, W, H, o, h_rgb, h_T, stream, async_=True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(K):
        ctx.gs_render_views_host(hs, my, W, H, o, h_rgb, h_T, stream, async_=True)
    e1.record(stream)
    e1.synchronize()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{tag}: events {e0.elapsed_time(e1):.2f} ms, wall to e1 {1e3*(t1-t0):.2f} ms, wall to device idle {1e3*(t2-t0):.2f} ms", flush=True)

e2e("fresh")
# an orbit with timing flags (the A/B section)
ctx.gs_render_views(st, my, W, H, opts(bg, sh_degree=3, flags=GS_FLAG_TIMING | GS_FLAG_OBOX), out_rgb, out_T, stream)
torch.cuda.synchronize(); ctx.gs_stage_times()
e2e("after timing orbit")
ctx.gs_render_views(st, my, W, H, opts(bg, sh_degree=3, blend=GS_BLEND_DIRECT, flags=GS_FLAG_TIMING | GS_FLAG_OBOX), out_rgb, out_T, stream)
torch.cuda.synchronize(); ctx.gs_stage_times()
e2e("after direct orbit")
ctx.gs_render_views(st, my, W, H, opts(bg, sh_degree=3, flags=GS_FLAG_TIMING | GS_FLAG_TIGHT), out_rgb, out_T, stream)
torch.cuda.synchronize(); ctx.gs_stage_times()
e2e("after tight orbit")
for nb in (1, 2, 4, 8):
    for k in range(nb):
        ctx.gs_render(st, my[0], W, H, opts(bg, sh_degree=3, flags=GS_FLAG_OBOX, band=k, n_bands=nb), out_rgb[0], out_T[0], stream)
torch.cuda.synchronize()
e2e("after row bands")
cs = [camera(c) for c in synth.orbit_cameras(64, W, H, math.radians(60.0))][::8]
r8 = torch.empty((8, 3, H, W), device="cuda"); t8 = torch.empty((8, H, W), device="cuda")
ctx.gs_render_views(st, cs, W, H, o, r8, t8, stream)
torch.cuda.synchronize()
e2e("after 8-view orbit")
