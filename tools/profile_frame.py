"""Renders a few C5 frames through the C-ABI (for ncu launch lists / --set full)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_02120_b200 import (GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC, Context, camera, opts,  # noqa: E402
                                   scene_to_device, synth)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--view", type=int, default=0)
ap.add_argument("--blend", default="tc", choices=["tc", "direct", "mma"])
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--obox", action="store_true")
ap.add_argument("--group", type=int, default=0, help="render views [view, view+group) with gs_render_views "
                "(one view-group preprocess launch, chains serialised on one stream) instead of gs_render")
a = ap.parse_args()
scene, cams, bg = synth.make_config(a.config, views=64 if a.config == "C5" else 1)
cam = cams[a.view % len(cams)]
ctx = Context(0, max_points=scene.n, max_keys=48 << 20, max_w=cam.W, max_h=cam.H)
st = scene_to_device(scene)
rgb = torch.empty((3, cam.H, cam.W), device="cuda")
T = torch.empty((cam.H, cam.W), device="cuda")
o = opts(bg, sh_degree=scene.sh_degree, batch=a.batch, flags=16 if a.obox else 0,
         blend={"tc": GS_BLEND_TC, "direct": GS_BLEND_DIRECT, "mma": GS_BLEND_MMA}[a.blend])
if a.group:
    ctx.gs_set_view_group(a.group, False)
    gc = [camera(cams[(a.view + j) % len(cams)]) for j in range(a.group)]
    grgb = torch.empty((a.group, 3, cam.H, cam.W), device="cuda")
    gT = torch.empty((a.group, cam.H, cam.W), device="cuda")
for _ in range(a.frames):
    if a.group:
        ctx.gs_render_views(st, gc, cam.W, cam.H, o, grgb, gT)
    else:
        ctx.gs_render(st, camera(cam), cam.W, cam.H, o, rgb, T)
torch.cuda.synchronize()
print("ok", ctx.gs_last_stats().n_keys)
