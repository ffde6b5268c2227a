"""Precision of the tensor-core exponent for the library in GS_RENDER_LIB (default
build: TF32 hi/lo, K = 16; a -DGS_BLEND_KSTEPS=1 variant: single TF32 pass, K = 8):
max |d ln alpha| over the oracle's kept pairs on sampled C2 tiles, and the C2 frame
against the oracle (max abs on unflagged pixels, pixels above 2e-3, PSNR)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from gpu_util import compare, gpu_render, make_ctx  # noqa: E402
from paper_2604_02120_b200 import synth  # noqa: E402

scene, cams, bg = synth.make_config("C2")
cam = cams[0]
ctx = make_ctx(scene, cam)
pre = oracle.preprocess(scene, cam)
b = oracle.binning(pre, cam.W, cam.H)
gx = (cam.W + 15) // 16
rng = np.random.default_rng(0)
ranges = np.zeros_like(b["ranges"])
sel = rng.choice(len(ranges), 64, replace=False)
ranges[sel] = b["ranges"][sel]
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
out_m = torch.full((b["K"], 256), float("nan"), device="cuda")
ctx.gs_debug_exponents(scene.n, t(pre["xy"]), t(pre["conic"]), t(pre["opacity"]), t(b["vals"].view(np.int32)),
                       b["K"], t(ranges.view(np.int32)), cam.W, cam.H, out_m)
m = out_m.cpu().numpy()
lanes = np.arange(256)
w, l = lanes // 32, lanes % 32
pxi, pyi = 8 * (w % 2) + l % 8, 4 * (w // 2) + l // 8
worst, n = 0.0, 0
for ts in sel:
    s, e = b["ranges"][ts]
    if e == s:
        continue
    px, py = 16 * (ts % gx) + pxi, 16 * (ts // gx) + pyi
    idx = b["vals"][s:e]
    xy, co, o = (pre[k][idx].astype(np.float64) for k in ("xy", "conic", "opacity"))
    dx, dy = xy[:, :1] - px[None], xy[:, 1:2] - py[None]
    ln_a = np.log(o)[:, None] - 0.5 * (co[:, :1] * dx * dx + co[:, 2:3] * dy * dy) - co[:, 1:2] * dx * dy
    keep = ln_a >= np.log(1 / 255.0)
    d = np.abs(m[s:e] * np.log(2.0) - ln_a)[keep]
    n += d.size
    worst = max(worst, float(d.max()) if d.size else 0.0)
rgb, T = gpu_render(ctx, scene, cam, bg)
_, _, ref = oracle.render(scene, cam, bg)
c = compare(rgb, T, ref)
print(f"lib={os.environ.get('GS_RENDER_LIB', 'default')} max|d ln alpha|={worst:.3e} over {n} kept pairs; "
      f"frame: max unflagged {c['max_unflagged']:.3e}, pixels > 2e-3: {c['n_over']} "
      f"({c['over_unflagged']} unflagged), PSNR {c['psnr']:.1f} dB")
