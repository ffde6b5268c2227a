"""Prints the per-stage timeline (GS_FLAG_TIMING spans) of one C5 orbit segment in the
bench's launch configuration (view groups, concurrent chains): which stage runs when."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2604_02120_b200 import GS_FLAG_OBOX, GS_FLAG_TIMING, Context, camera, opts, scene_to_device, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=32)
ap.add_argument("--serial", action="store_true")
ap.add_argument("--group", type=int, default=16)
a = ap.parse_args()
scene, cams, bg = synth.make_config("C5", views=64)
cam = cams[0]
ctx = Context(0, max_points=scene.n, max_keys=48 << 20, max_w=cam.W, max_h=cam.H)
ctx.gs_set_view_group(a.group, not a.serial)
st = scene_to_device(scene)
cs = [camera(c) for c in cams[:a.views]]
rgb = torch.empty((a.views, 3, cam.H, cam.W), device="cuda")
T = torch.empty((a.views, cam.H, cam.W), device="cuda")
o = opts(bg, sh_degree=scene.sh_degree, flags=GS_FLAG_TIMING | GS_FLAG_OBOX)
for _ in range(2):
    ctx.gs_render_views(st, cs, cam.W, cam.H, o, rgb, T)
torch.cuda.synchronize()
ctx.gs_stage_times()
ctx.gs_render_views(st, cs, cam.W, cam.H, o, rgb, T)
torch.cuda.synchronize()
names = ("pre", "bin", "blend")
tl = ctx.gs_debug_timeline()
t_end = max(t1 for _, _, t1 in tl)
for stg, t0, t1 in sorted(tl, key=lambda x: x[1]):
    print(f"{names[stg]:6s} {t0:8.3f} {t1:8.3f}  {t1 - t0:7.3f}  " + " " * int(t0 / t_end * 60) + "#" * max(1, int((t1 - t0) / t_end * 60)))
print(f"total {t_end:.3f} ms for {a.views} views = {t_end / a.views:.3f} ms/view")
