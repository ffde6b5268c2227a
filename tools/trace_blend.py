"""Per-batch timeline of the tensor-core blend (CTA 0) on a C5 view, from gs_debug_set_trace."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_02120_b200 import Context, camera, opts, scene_to_device, synth  # noqa: E402

scene, cams, bg = synth.make_config("C5", views=64)
cam = cams[0]
ctx = Context(0, max_points=scene.n, max_keys=48 << 20, max_w=cam.W, max_h=cam.H)
st = scene_to_device(scene)
rgb = torch.empty((3, cam.H, cam.W), device="cuda")
T = torch.empty((cam.H, cam.W), device="cuda")
o = opts(bg, sh_degree=3)
ctx.gs_render(st, camera(cam), cam.W, cam.H, o, rgb, T)
tr = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
ctx.gs_debug_set_trace(tr)
ctx.gs_render(st, camera(cam), cam.W, cam.H, o, rgb, T)
torch.cuda.synchronize()
ctx.gs_debug_set_trace(None)
t = tr.cpu().numpy().reshape(1024, 16).astype(np.float64)
valid = t[:, 7] > 0
t0 = t[valid][:, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10]].min()
names = ["push0", "push1", "bgot", "bfree", "bdone", "mrows", "missue", "c0beg", "c0end", "c7beg", "c7end"]
print("batch " + " ".join(f"{n:>7}" for n in names) + "   (cycles since first event)")
for b in range(0, 1024):
    if not valid[b]:
        continue
    if b < 40 or b % 50 == 0:
        print(f"{b:5d} " + " ".join(f"{(t[b, e] - t0) if t[b, e] > 0 else -1:7.0f}" for e in range(11)))
nb = int(valid.sum())
c = t[valid]
span = c[:, 8].max() - c[:, 7].min()
print(f"batches {nb}, span {span:.0f} cyc, {span / nb:.0f} cyc/batch")
for a, bb, label in [(0, 1, "producer raw_empty wait"), (2, 3, "builder stage-free wait"), (3, 4, "builder build"),
                     (5, 6, "MMA empty wait"), (7, 8, "compositor w0 work"), (9, 10, "compositor w7 work")]:
    d = c[:, bb] - c[:, a]
    d = d[(c[:, a] > 0) & (c[:, bb] > 0)]
    print(f"{label:28s} mean {d.mean():8.0f}  median {np.median(d):8.0f} cyc")
d = c[1:, 7] - c[:-1, 8]
print(f"{'compositor w0 idle (wait)':28s} mean {d.mean():8.0f}  median {np.median(d):8.0f} cyc")
d = c[:, 7] - c[:, 6]
print(f"{'MMA issue -> compositor beg':28s} mean {d.mean():8.0f}  median {np.median(d):8.0f} cyc")
d = c[:, 5] - c[:, 4]
print(f"{'builder done -> MMA rows':28s} mean {d.mean():8.0f}  median {np.median(d):8.0f} cyc")
