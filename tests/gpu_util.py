"""Helpers for the -m gpu parity tests: run the CUDA path through the C-ABI and
compare it with the oracle on the same seeded inputs."""
import numpy as np

import oracle
from paper_2604_02120_b200 import Context, camera, opts, scene_to_device, synth

MAX_ABS = 2e-3      # per channel, on pixels the oracle does not flag (BASELINE.json north_star)
MIN_PSNR = 50.0     # dB over all pixels


def make_ctx(scene, cam, max_keys=None):
    return Context(0, max_points=max(scene.n, 1), max_keys=max_keys or (1 << 24), max_w=cam.W, max_h=cam.H)


def _sh_opts(scene, **kw):
    """opts() for a scene whose SH record may be longer than its degree needs (stride =
    record length) or hold plain colours (degree -1, shs [N,3])."""
    stride = scene.shs.shape[1] if scene.shs.ndim == 3 else 1
    return opts(sh_degree=scene.sh_degree, sh_stride=stride, **kw)


def gpu_preprocess(ctx, scene, cam, st=None, flags=0, scale_modifier=1.0):
    import torch
    st = st or scene_to_device(scene)
    n = scene.n
    dev = "cuda"
    outs = dict(depth=torch.empty(n, device=dev), xy=torch.empty((n, 2), device=dev),
                conic=torch.empty((n, 3), device=dev), rgb=torch.empty((n, 3), device=dev),
                rect=torch.empty((n, 4), dtype=torch.int32, device=dev),
                radius=torch.empty(n, dtype=torch.int32, device=dev),
                touched=torch.empty(n, dtype=torch.int32, device=dev))
    ctx.gs_debug_preprocess(st, camera(cam), cam.W, cam.H,
                            _sh_opts(scene, flags=flags, scale_modifier=scale_modifier), outs)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in outs.items()}
    out["touched"] = out["touched"].view(np.uint32)
    return out


def gpu_binning(ctx, scene, cam, capacity=None, st=None, flags=0, scale_modifier=1.0):
    import torch
    st = st or scene_to_device(scene)
    cap = capacity or (1 << 22)
    keys = torch.empty(cap, dtype=torch.int64, device="cuda")
    vals = torch.empty(cap, dtype=torch.int32, device="cuda")
    ntiles = ((cam.W + 15) // 16) * ((cam.H + 15) // 16)
    ranges = torch.empty((ntiles, 2), dtype=torch.int32, device="cuda")
    code, K = ctx.gs_debug_binning(st, camera(cam), cam.W, cam.H,
                                   _sh_opts(scene, flags=flags, scale_modifier=scale_modifier), keys, vals, ranges)
    if code != 0:
        return code, K, None
    return code, K, dict(keys=keys[:K].cpu().numpy().view(np.uint64), vals=vals[:K].cpu().numpy().view(np.uint32),
                         ranges=ranges.cpu().numpy().view(np.uint32))


def gpu_render(ctx, scene, cam, bg, blend=0, st=None, flags=0, scale_modifier=1.0):
    import torch
    st = st or scene_to_device(scene)
    out_rgb = torch.full((3, cam.H, cam.W), float("nan"), device="cuda")
    out_T = torch.full((cam.H, cam.W), float("nan"), device="cuda")
    ctx.gs_render(st, camera(cam), cam.W, cam.H,
                  _sh_opts(scene, bg=bg, blend=blend, flags=1 | flags, scale_modifier=scale_modifier), out_rgb, out_T)
    torch.cuda.synchronize()
    return out_rgb.cpu().numpy().astype(np.float64), out_T.cpu().numpy().astype(np.float64)


def gpu_blend_from(ctx, pre, binned, W, H, bg, blend=0):
    """Stage (d) alone on oracle-produced splats and binning (test harness upload)."""
    import torch
    t = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    n = pre["xy"].shape[0]
    vals = binned["vals"] if binned["K"] > 0 else np.zeros(1, np.uint32)
    out_rgb = torch.full((3, H, W), float("nan"), device="cuda")
    out_T = torch.full((H, W), float("nan"), device="cuda")
    ctx.gs_debug_blend(n, t(pre["xy"]), t(pre["conic"]), t(pre["opacity"]), t(pre["rgb"]),
                       t(vals.view(np.int32)), binned["K"], t(binned["ranges"].view(np.int32)), W, H,
                       opts(bg, blend=blend, flags=1), out_rgb, out_T)
    torch.cuda.synchronize()
    return out_rgb.cpu().numpy().astype(np.float64), out_T.cpu().numpy().astype(np.float64)


def compare(rgb, T, ref):
    err = np.abs(rgb - ref["rgb"])
    flag = ref["flag"]
    ok = ~flag
    mse = float((err ** 2).mean())
    psnr = 10 * np.log10(1.0 / max(mse, 1e-30))
    over = (err.max(0) > MAX_ABS)
    return dict(max_unflagged=float(err[:, ok].max()) if ok.any() else 0.0, max_all=float(err.max()),
                n_over=int(over.sum()), over_unflagged=int((over & ok).sum()), psnr=psnr,
                flagged=float(flag.mean()), T_max=float(np.abs(T - ref["T"])[ok].max()) if ok.any() else 0.0,
                over_within_bound=bool(np.all(err.max(0)[over] <= ref["bound"][over] + MAX_ABS)))
