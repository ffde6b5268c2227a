"""compute-sanitizer driver (race / memory checking of the hot path).

Runs the render path through the C-ABI on small seeded cases so that
`compute-sanitizer --tool {memcheck,synccheck,initcheck,racecheck}` can watch
every kernel: the four blends (tcgen05 mbarrier/TMEM pipeline with the supertile
list filter and the TMA frame store, its colour-MMA variant, mma.sync, CUDA-core
direct), both intersection modes, the binning chains (supertile, two-level and
one-level), a concurrent view group and the asynchronous host entry point.

    compute-sanitizer --tool memcheck python tests/sanitize_cases.py [--quick]

Prints one line per render and exits non-zero if any frame has a non-finite
pixel; the sanitizer's own exit code reports its findings (--error-exitcode).
Imports no oracle: frames are only checked for finiteness and tc-vs-direct
closeness here (parity proper is tests/test_gpu_parity.py).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

from cases import CASES  # noqa: E402
from paper_2604_02120_b200 import (GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC, GS_BLEND_TC_COLOR,  # noqa: E402
                                   GS_FLAG_OBOX, Context, camera, opts, scene_to_device, scene_to_host, synth)

BLENDS = {"tc": GS_BLEND_TC, "mma": GS_BLEND_MMA, "direct": GS_BLEND_DIRECT, "tc_color": GS_BLEND_TC_COLOR}


def _opts(scene, bg, blend, flags, batch=0):
    stride = scene.shs.shape[1] if scene.shs.ndim == 3 else 1
    return opts(bg, sh_degree=scene.sh_degree, sh_stride=stride, blend=blend, flags=1 | flags, batch=batch)


def render(ctx, st, scene, cam, bg, blend, flags, batch=0):
    rgb = torch.empty((3, cam.H, cam.W), device="cuda")
    T = torch.empty((cam.H, cam.W), device="cuda")
    ctx.gs_render(st, camera(cam), cam.W, cam.H, _opts(scene, bg, blend, flags, batch), rgb, T)
    torch.cuda.synchronize()
    return rgb.cpu().numpy(), T.cpu().numpy()


def main(quick=False):
    bad = 0
    names = ["C1", "ragged", "adversarial"] + ([] if quick else ["dense", "tall"])
    for name in names:
        scene, cam, bg = CASES[name]()
        ctx = Context(0, max_points=max(scene.n, 1), max_keys=1 << 22, max_w=cam.W, max_h=cam.H)
        st = scene_to_device(scene)
        frames = {}
        for flags, fname in ((0, "rect"), (GS_FLAG_OBOX, "obox")):
            for bname, b in BLENDS.items():
                rgb, T = render(ctx, st, scene, cam, bg, b, flags, batch=64 if b == GS_BLEND_MMA else 0)
                ok = np.isfinite(rgb).all() and np.isfinite(T).all()
                bad += not ok
                frames[(fname, bname)] = rgb
                print(f"{name:12s} {fname:5s} {bname:7s} finite={ok} mean={rgb.mean():.5f}", flush=True)
        d = np.abs(frames[("obox", "tc")] - frames[("rect", "direct")]).max()
        print(f"{name:12s} max|tc(obox) - direct(rect)| = {d:.2e}", flush=True)
        ctx.close()

    # a concurrent view group (per-view workspaces, context streams, slot sets) and the
    # asynchronous host entry point (staging buffers, per-frame D2H)
    scene, cams, bg = synth.make_config("C2", n_override=20000, views=5)
    W, H = 200, 150
    cams = synth.orbit_cameras(5, W, H, 0.8)
    ctx = Context(0, max_points=scene.n, max_keys=1 << 22, max_w=W, max_h=H)
    ctx.gs_set_view_group(2, True)
    st = scene_to_device(scene)
    o = _opts(scene, bg, GS_BLEND_TC, GS_FLAG_OBOX)
    rgb = torch.empty((5, 3, H, W), device="cuda")
    T = torch.empty((5, H, W), device="cuda")
    ctx.gs_render_views(st, [camera(c) for c in cams], W, H, o, rgb, T)
    torch.cuda.synchronize()
    ok = bool(torch.isfinite(rgb).all() and torch.isfinite(T).all())
    bad += not ok
    print(f"view group (5 views, groups of 2, concurrent) finite={ok}", flush=True)
    sh = scene_to_host(scene)
    h_rgb = torch.empty((5, 3, H, W)).pin_memory()
    h_T = torch.empty((5, H, W)).pin_memory()
    for async_ in (False, True):
        ctx.gs_render_views_host(sh, [camera(c) for c in cams], W, H, o, h_rgb, h_T, async_=async_)
        torch.cuda.synchronize()
        same = bool(torch.equal(h_rgb, rgb.cpu()) and torch.equal(h_T, T.cpu()))
        bad += not same
        print(f"host entry point async={async_} equal to device frames={same}", flush=True)
    ctx.close()
    print("SANITIZE_CASES_DONE bad=%d" % bad, flush=True)
    return bad


if __name__ == "__main__":
    sys.exit(1 if main(quick="--quick" in sys.argv) else 0)
