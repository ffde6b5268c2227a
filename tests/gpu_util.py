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


def gpu_binning(ctx, scene, cam, capacity=None, st=None, flags=0, scale_modifier=1.0, blend=0):
    """Keys / values / ranges per tile. blend=GS_BLEND_TC (0, the default) bins into the
    supertile lists the tcgen05 blend filters (grids up to 512 supertiles; the library then
    derives the per-tile lists with the blend's own mask filter); the other blends take the
    per-tile two-level (or one-level) binning."""
    import torch
    st = st or scene_to_device(scene)
    cap = capacity or (1 << 22)
    keys = torch.empty(cap, dtype=torch.int64, device="cuda")
    vals = torch.empty(cap, dtype=torch.int32, device="cuda")
    ntiles = ((cam.W + 15) // 16) * ((cam.H + 15) // 16)
    ranges = torch.empty((ntiles, 2), dtype=torch.int32, device="cuda")
    code, K = ctx.gs_debug_binning(st, camera(cam), cam.W, cam.H,
                                   _sh_opts(scene, flags=flags, scale_modifier=scale_modifier, blend=blend), keys, vals,
                                   ranges)
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


MAX_FLAGGED = 0.01   # the margin mask may excuse at most 1 % of a frame's pixels


def compare(rgb, T, ref):
    """The pixel gate of SURVEY 8 gate 2: max |d| per channel on unflagged pixels, PSNR over
    all pixels, and (always reported) the all-pixel max |d| and the count of pixels above
    2e-3, each of which must be flagged and within its flip bound."""
    err = np.abs(rgb - ref["rgb"])
    flag = ref["flag"]
    ok = ~flag
    mse = float((err ** 2).mean())
    psnr = 10 * np.log10(1.0 / max(mse, 1e-30))
    over = (err.max(0) > MAX_ABS)
    return dict(max_unflagged=float(err[:, ok].max()) if ok.any() else 0.0, max_all=float(err.max()),
                n_over=int(over.sum()), over_unflagged=int((over & ok).sum()), psnr=psnr,
                flagged=float(flag.mean()), n_flagged=int(flag.sum()), n_pixels=int(flag.size),
                T_max=float(np.abs(T - ref["T"])[ok].max()) if ok.any() else 0.0,
                T_max_all=float(np.abs(T - ref["T"]).max()),
                over_within_bound=bool(np.all(err.max(0)[over] <= ref["bound"][over] + MAX_ABS)))


def check_frame(case, rgb, T, ref, check_T=True):
    """compare() and every assertion of the pixel gate; the row is appended to the file named
    by $GS_PARITY_LOG (JSON lines; tools/parity_table.py turns it into the committed table)."""
    import json
    import os
    m = compare(rgb, T, ref)
    m["case"] = case
    log = os.environ.get("GS_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps(m) + "\n")
    assert m["max_unflagged"] <= MAX_ABS, m
    assert m["psnr"] >= MIN_PSNR, m
    assert m["over_unflagged"] == 0, m                 # every pixel above 2e-3 is flagged ...
    assert m["over_within_bound"], m                   # ... and within its flip bound
    assert m["max_all"] <= MAX_ABS + float(ref["bound"].max()), m
    assert m["flagged"] <= MAX_FLAGGED, m
    if check_T:
        assert m["T_max"] <= MAX_ABS, m
    return m


def tile_pixels(tile, gx):
    """Pixel coordinates of the 256 compositor lanes of `tile` (k_blend_tc's lane layout:
    warp w covers the 8x4 block at (8 (w % 2), 4 (w / 2)))."""
    lanes = np.arange(256)
    w, l = lanes // 32, lanes % 32
    return 16 * (tile % gx) + 8 * (w % 2) + l % 8, 16 * (tile // gx) + 4 * (w // 2) + l // 8


def exponent_errors(ctx, n, pre, binned, W, H, tiles):
    """Raw tensor-core exponents (gs_debug_exponents: log2 alpha as the MMA left it in TMEM)
    of the oracle's lists on `tiles`, against the float64 ln alpha of Eq. (3) from the same
    fp32 splats. Returns, over the pairs the oracle keeps (alpha >= 1/255), the error
    |d ln alpha| and the magnitude S of the Eq. (6) terms the GEMM adds up (sum of
    |v_k p_k| over the tile-centre expansion, reading R-6, plus the magnitudes of the
    three products inside v_5 and |ln o|): the scale of fp32/TF32 rounding in the sum."""
    import torch
    gx = (W + 15) // 16
    ranges = np.zeros_like(binned["ranges"])
    ranges[tiles] = binned["ranges"][tiles]
    K = binned["K"]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out_m = torch.full((max(K, 1), 256), float("nan"), device="cuda")
    ctx.gs_debug_exponents(n, t(pre["xy"]), t(pre["conic"]), t(pre["opacity"]), t(binned["vals"].view(np.int32)),
                           K, t(ranges.view(np.int32)), W, H, out_m)
    m = out_m.cpu().numpy()
    errs, mags = [], []
    for tile in tiles:
        s, e = binned["ranges"][tile]
        if e == s:
            continue
        px, py = tile_pixels(tile, gx)
        idx = binned["vals"][s:e]
        xy = pre["xy"][idx].astype(np.float64)
        co = pre["conic"][idx].astype(np.float64)
        o = pre["opacity"][idx].astype(np.float64)
        A, B, C = co[:, 0:1], co[:, 1:2], co[:, 2:3]
        dx = xy[:, 0:1] - px[None, :]
        dy = xy[:, 1:2] - py[None, :]
        ln_a = np.log(o)[:, None] - 0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy
        keep = ln_a >= np.log(1 / 255.0)
        xc, yc = 16.0 * (tile % gx) + 7.5, 16.0 * (tile // gx) + 7.5
        xh, yh = xy[:, 0:1] - xc, xy[:, 1:2] - yc
        xb, yb = xc - px[None, :], yc - py[None, :]
        S = (0.5 * np.abs(A) * xb * xb + 0.5 * np.abs(C) * yb * yb + np.abs(B * xb * yb)
             + np.abs(A * xh + B * yh) * np.abs(xb) + np.abs(C * yh + B * xh) * np.abs(yb)
             + 0.5 * np.abs(A) * xh * xh + 0.5 * np.abs(C) * yh * yh + np.abs(B * xh * yh)
             + np.abs(np.log(o))[:, None])
        errs.append(np.abs(m[s:e] * np.log(2.0) - ln_a)[keep])
        mags.append(S[keep])
    if not errs:
        return np.zeros(0), np.zeros(0)
    return np.concatenate(errs), np.concatenate(mags)
