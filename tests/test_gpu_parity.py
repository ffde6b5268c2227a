"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * preprocess outputs, sorted keys, values and tile ranges: bit-exact;
  * pixels: max |d| <= 2e-3 per channel on pixels the oracle does not flag as
    decision-ambiguous (margin mask, reading R-21), PSNR >= 50 dB over all
    pixels; every pixel above 2e-3 must be flagged and within its flip bound.
"""
import numpy as np
import pytest

import oracle
from paper_2604_02120_b200 import GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC, GS_BLEND_TC_COLOR, GsError, synth

from cases import CASES, _adversarial, _cfg, _dense, _ragged, _wide  # noqa: F401
from gpu_util import (MAX_ABS, MIN_PSNR, check_frame, exponent_errors, gpu_binning, gpu_blend_from, gpu_preprocess,
                      gpu_render, make_ctx)

pytestmark = pytest.mark.gpu

BIT_EXACT_KEYS = ("depth", "xy", "conic", "rgb", "rect", "radius", "touched")


@pytest.mark.parametrize("case", list(CASES))
def test_preprocess_bit_exact(case):
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    got = gpu_preprocess(ctx, scene, cam)
    ref = oracle.preprocess(scene, cam)
    assert (ref["touched"] > 0).sum() > 0
    for k in BIT_EXACT_KEYS:
        a, b = got[k], ref[k]
        a = a.view(np.uint32) if a.dtype == np.float32 else a.astype(np.int64)
        b = b.view(np.uint32) if b.dtype == np.float32 else b.astype(np.int64)
        bad = np.nonzero((a != b).reshape(len(a), -1).any(1))[0]
        assert len(bad) == 0, f"{k}: {len(bad)} Gaussians differ, first {bad[:5]}"


@pytest.mark.parametrize("lists", [GS_BLEND_TC, GS_BLEND_MMA], ids=["supertile", "per_tile"])
@pytest.mark.parametrize("case", list(CASES))
def test_binning_bit_exact(case, lists):
    """Both binnings: the supertile lists of the tcgen05 blend (filtered per tile by the
    mask bits) and the per-tile two-level / one-level lists of the other blends."""
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    code, K, got = gpu_binning(ctx, scene, cam, blend=lists)
    assert code == 0
    pre = oracle.preprocess(scene, cam)
    ref = oracle.binning(pre, cam.W, cam.H)
    assert K == ref["K"]
    assert np.array_equal(got["keys"], ref["keys"])
    assert np.array_equal(got["vals"], ref["vals"])
    assert np.array_equal(got["ranges"], ref["ranges"])


@pytest.mark.parametrize("blend", [GS_BLEND_TC, GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC_COLOR],
                         ids=["tc", "direct", "mma", "tc_color"])
@pytest.mark.parametrize("case", list(CASES))
def test_blend_parity_on_oracle_binning(case, blend):
    """Stage (d) alone: oracle splats + oracle binning uploaded by the harness."""
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    pre, b, ref = oracle.render(scene, cam, bg)
    rgb, T = gpu_blend_from(ctx, pre, b, cam.W, cam.H, bg, blend)
    check_frame(f"blend_only/{case}/{['tc', 'direct', 'mma', 'tc_color'][blend]}", rgb, T, ref)


@pytest.mark.parametrize("blend", [GS_BLEND_TC, GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC_COLOR],
                         ids=["tc", "direct", "mma", "tc_color"])
@pytest.mark.parametrize("case", list(CASES))
def test_render_parity_end_to_end(case, blend):
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    rgb, T = gpu_render(ctx, scene, cam, bg, blend)
    assert np.isfinite(rgb).all() and np.isfinite(T).all()
    _, _, ref = oracle.render(scene, cam, bg)
    check_frame(f"end_to_end/{case}/{['tc', 'direct', 'mma', 'tc_color'][blend]}", rgb, T, ref)


@pytest.mark.parametrize("case", list(CASES))
def test_exponent_precision_bound(case):
    """|d ln alpha| of the tensor-core exponent (TF32 hi/lo, reading R-11) stays below the
    bound the margin mask assumes, delta = DELTA_0 + EPS_REL * S (S = magnitude of the
    Eq. (6) terms about the tile centre), on every pair the oracle keeps: every tile of the
    small cases, 96 sampled tiles of the large ones; the adversarial case has needles with
    anisotropy up to 300 (SURVEY C-11)."""
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    pre = oracle.preprocess(scene, cam)
    b = oracle.binning(pre, cam.W, cam.H)
    nt = len(b["ranges"])
    tiles = np.arange(nt) if nt <= 200 else np.random.default_rng(0).choice(nt, 96, replace=False)
    err, S = exponent_errors(ctx, scene.n, pre, b, cam.W, cam.H, tiles)
    bound = oracle.DELTA_0 + oracle.EPS_REL * S
    print(f"{case}: max |d ln alpha| = {err.max():.3e}, max err/bound = {(err / bound).max():.3f} "
          f"over {err.size} kept pairs")
    assert err.size > 1000
    assert (err <= bound).all(), (float(err.max()), float((err / bound).max()))


def test_determinism_and_tc_vs_direct():
    scene, cam, bg = _cfg("C2")
    ctx = make_ctx(scene, cam)
    a, ta = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC)
    b, tb = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC)
    assert np.array_equal(a, b) and np.array_equal(ta, tb)
    c, _ = gpu_render(ctx, scene, cam, bg, GS_BLEND_DIRECT)
    assert 10 * np.log10(1 / max(((a - c) ** 2).mean(), 1e-30)) >= MIN_PSNR


def test_empty_scene_is_background():
    scene = synth.object_scene(0, 0, sh_degree=0)
    cam = synth.look_at((0, 0, -4), (0, 0, 0), 40, 24, 0.7)
    ctx = make_ctx(scene, cam, max_keys=1024)
    rgb, T = gpu_render(ctx, scene, cam, (0.1, 0.2, 0.3))
    for ch, v in enumerate((0.1, 0.2, 0.3)):
        assert (rgb[ch] == np.float32(v)).all()
    assert (T == 1.0).all()


def test_all_culled_scene_is_background():
    scene = synth.object_scene(500, 3, sh_degree=1)
    scene.means[:] = np.array([0, 0, -10], np.float32)        # behind the camera at z=-4
    cam = synth.look_at((0, 0, -4), (0, 0, 0), 48, 48, 0.7)
    ctx = make_ctx(scene, cam, max_keys=1024)
    rgb, T = gpu_render(ctx, scene, cam, (0.5, 0.5, 0.5))
    assert (rgb == np.float32(0.5)).all() and (T == 1.0).all()


def test_capacity_error_is_reported_not_truncated():
    scene, cam, bg = _cfg("C1")
    ctx = make_ctx(scene, cam, max_keys=100)
    with pytest.raises(GsError) as e:
        gpu_render(ctx, scene, cam, bg)
    assert e.value.code == -3
    st = ctx.gs_last_stats()
    assert st.n_keys == oracle.binning(oracle.preprocess(scene, cam), cam.W, cam.H)["K"]


@pytest.mark.slow
@pytest.mark.parametrize("obox", [False, True], ids=["vanilla", "obox"])
def test_full_size_c5_view_sampled_parity(obox):
    """BASELINE.json configs[4] shape at full size (6M Gaussians, 1920x1080) in the
    launch configuration bench.py times (gs_render_views, view group of 4, concurrent
    binning chains; vanilla rect and GS_FLAG_OBOX): preprocess and binning bit-exact
    over everything; the orbit's frame equals the single-view frame bit for bit;
    pixels on 48 sampled tiles against the oracle."""
    import torch
    from paper_2604_02120_b200 import GS_FLAG_OBOX, Context, camera, opts, scene_to_device
    flags = GS_FLAG_OBOX if obox else 0
    scene, cams, bg = synth.make_config("C5", views=64)
    cam = cams[0]
    ctx = Context(0, max_points=scene.n, max_keys=64 << 20, max_w=cam.W, max_h=cam.H)
    st = scene_to_device(scene)
    got = gpu_preprocess(ctx, scene, cam, st, flags=flags)
    pre = oracle.preprocess(scene, cam, obox=obox)
    for k in BIT_EXACT_KEYS:
        a = got[k].view(np.uint32) if got[k].dtype == np.float32 else got[k].astype(np.int64)
        b = pre[k].view(np.uint32) if pre[k].dtype == np.float32 else pre[k].astype(np.int64)
        vis = pre["touched"] > 0
        assert np.array_equal(a[vis], b[vis]) and np.array_equal(got["touched"], pre["touched"]), k
    code, K, gb = gpu_binning(ctx, scene, cam, capacity=64 << 20, st=st, flags=flags)
    assert code == 0
    ref_b = oracle.binning(pre, cam.W, cam.H)
    assert K == ref_b["K"]
    assert np.array_equal(gb["keys"], ref_b["keys"]) and np.array_equal(gb["vals"], ref_b["vals"])
    assert np.array_equal(gb["ranges"], ref_b["ranges"])
    rgb, T = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, st=st, flags=flags)
    # the bench's path: views in one group of up to 16, chains concurrent; view 0 must match
    ctx.gs_set_view_group(16, True)
    orgb = torch.empty((6, 3, cam.H, cam.W), device="cuda")
    oT = torch.empty((6, cam.H, cam.W), device="cuda")
    ctx.gs_render_views(st, [camera(c) for c in cams[:6]], cam.W, cam.H,
                        opts(bg, sh_degree=scene.sh_degree, flags=flags), orgb, oT)
    torch.cuda.synchronize()
    assert np.array_equal(orgb[0].cpu().numpy().astype(np.float64), rgb)
    assert np.array_equal(oT[0].cpu().numpy().astype(np.float64), T)
    rng = np.random.default_rng(7)
    ntiles = len(ref_b["ranges"])
    sel = rng.choice(ntiles, 48, replace=False)
    r2 = np.zeros_like(ref_b["ranges"])
    r2[sel] = ref_b["ranges"][sel]
    b2 = dict(ref_b); b2["ranges"] = r2
    ref = oracle.blend(pre, b2, cam.W, cam.H, bg)
    gx = (cam.W + 15) // 16
    mask = np.zeros((cam.H, cam.W), bool)
    for t in sel:
        mask[16 * (t // gx):16 * (t // gx) + 16, 16 * (t % gx):16 * (t % gx) + 16] = True
    sub = {k: ref[k][..., mask] for k in ("rgb", "T", "flag", "bound")}
    check_frame(f"C5_full/{'obox' if obox else 'vanilla'}/48_tiles", rgb[:, mask], T[mask], sub)


# ---------------------------------------------------------------------------
# N3: tile-exact intersection (GS_FLAG_TIGHT)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", list(CASES))
def test_tight_intersection_renders_bit_identical(case):
    """Dropped pairs are alpha-skipped anyway and every exponent is independent of
    the batch it lands in, so the frame is bit-identical to the vanilla-rect one."""
    from paper_2604_02120_b200 import GS_FLAG_TIGHT
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    a, ta = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC)
    b, tb = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, flags=GS_FLAG_TIGHT)
    assert np.array_equal(a, b) and np.array_equal(ta, tb)


@pytest.mark.parametrize("case", ["C1", "C2", "adversarial"])
def test_tight_binning_is_an_alpha_exact_subset(case):
    """Tight lists = the vanilla lists minus pairs whose alpha < 1/255 on every
    pixel of the tile (checked by brute force in float64 against the oracle's
    splats); the per-tile order is the vanilla order."""
    from paper_2604_02120_b200 import GS_FLAG_TIGHT
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    code, K, tb = gpu_binning(ctx, scene, cam, flags=GS_FLAG_TIGHT)
    assert code == 0
    pre = oracle.preprocess(scene, cam)
    ref = oracle.binning(pre, cam.W, cam.H)
    assert 0 < K < ref["K"]
    gx = (cam.W + 15) // 16
    rng = np.random.default_rng(0)
    tiles = np.nonzero(ref["ranges"][:, 1] > ref["ranges"][:, 0])[0]
    for t in rng.choice(tiles, min(60, len(tiles)), replace=False):
        v_all = ref["vals"][ref["ranges"][t, 0]:ref["ranges"][t, 1]]
        v_t = tb["vals"][tb["ranges"][t, 0]:tb["ranges"][t, 1]] if tb["ranges"][t, 1] > tb["ranges"][t, 0] else []
        kept = set(int(v) for v in v_t)
        assert [int(v) for v in v_all if int(v) in kept] == [int(v) for v in v_t]    # order preserved
        tx, ty = t % gx, t // gx
        yy, xx = np.mgrid[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16]
        inside = (xx < cam.W) & (yy < cam.H)
        for i in v_all:
            if int(i) in kept:
                continue
            dx = float(pre["xy"][i, 0]) - xx[inside]
            dy = float(pre["xy"][i, 1]) - yy[inside]
            A, B, C = (float(c) for c in pre["conic"][i])
            a = float(pre["opacity"][i]) * np.exp(-0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy)
            assert a.max() < 1.0 / 255.0, (t, i, a.max())


@pytest.mark.parametrize("flags", [0, 8, 16 | 32])
def test_view_groups_are_bit_identical_to_single_views(flags):
    """gs_render_views reads the scene once per view group (k_preprocess over up to 4
    views); every frame must equal the single-view gs_render of the same camera, for
    every group size, with a group count that does not divide the view count, and
    through the host-buffer entry point (copies overlapped on a second stream)."""
    import torch
    from paper_2604_02120_b200 import Context, camera, opts, scene_to_device, scene_to_host
    scene = synth.unbounded_scene(60000, 108, sh_degree=3)
    cams = synth.orbit_cameras(7, 320, 200, 1.0)
    bg = np.array([0.1, 0.2, 0.3], np.float32)
    ctx = Context(0, max_points=scene.n, max_keys=1 << 22, max_w=320, max_h=200)
    st = scene_to_device(scene)
    o = opts(bg, sh_degree=scene.sh_degree, flags=flags)
    ref_rgb, ref_T = [], []
    for cam in cams:
        r = torch.empty((3, cam.H, cam.W), device="cuda")
        t = torch.empty((cam.H, cam.W), device="cuda")
        ctx.gs_render(st, camera(cam), cam.W, cam.H, o, r, t)
        ref_rgb.append(r.cpu().numpy())
        ref_T.append(t.cpu().numpy())
    ref_rgb, ref_T = np.stack(ref_rgb), np.stack(ref_T)
    for g, conc in ((1, True), (2, True), (3, False), (3, True), (4, False), (4, True), (5, True), (16, True)):
        ctx.gs_set_view_group(g, conc)
        r = torch.full((7, 3, 200, 320), float("nan"), device="cuda")
        t = torch.full((7, 200, 320), float("nan"), device="cuda")
        ctx.gs_render_views(st, [camera(c) for c in cams], 320, 200, o, r, t)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), ref_rgb), g
        assert np.array_equal(t.cpu().numpy(), ref_T), g
        hr = torch.full((7, 3, 200, 320), float("nan")).pin_memory()
        ht = torch.full((7, 200, 320), float("nan")).pin_memory()
        ctx.gs_render_views_host(scene_to_host(scene), [camera(c) for c in cams], 320, 200, o, hr, ht)
        assert np.array_equal(hr.numpy(), ref_rgb), g
        assert np.array_equal(ht.numpy(), ref_T), g
    ctx.close()


@pytest.mark.parametrize("variant", ["sh0", "sh2_scale", "looking_away", "plain_colours"])
def test_compacted_view_group_preprocess_matches_single_views(variant):
    """View groups use the compacted preprocess (k_preprocess_cv: (Gaussian, view) pairs
    filtered by a conservative bound, then projected 32 per round by any lane); frames must
    equal the single-view kernel's bit for bit: SH degree 0 and 2 (the scalar SH-load path,
    stride 9), a scale modifier, a group whose cameras mostly look away from the scene (empty
    candidate lists) and plain colours (sh_degree -1)."""
    import torch
    from paper_2604_02120_b200 import Context, camera, opts, scene_to_device
    deg = {"sh0": 0, "sh2_scale": 2, "looking_away": 1, "plain_colours": 0}[variant]
    scene = synth.unbounded_scene(40000 + 77, 109, sh_degree=deg)
    sm = 1.7 if variant == "sh2_scale" else 1.0
    if variant == "plain_colours":
        scene.shs = np.ascontiguousarray(scene.shs[:, 0, :] * 0.28 + 0.5, np.float32)
        deg = -1
    cams = synth.orbit_cameras(9, 256, 144, 1.1)
    if variant == "looking_away":   # 7 of 9 cameras look outwards, away from the dense centre
        cams = [cams[0]] + [synth.look_at(tuple(np.array(c.campos, np.float64) * 1.0), tuple(
            np.array(c.campos, np.float64) * 3.0), 256, 144, 1.1) for c in cams[1:8]] + [cams[8]]
    bg = np.array([0.2, 0.1, 0.0], np.float32)
    ctx = Context(0, max_points=scene.n, max_keys=1 << 21, max_w=256, max_h=144)
    st = scene_to_device(scene)
    o = opts(bg, sh_degree=deg, sh_stride=(1 if deg < 0 else None), scale_modifier=sm, flags=16)
    ref_rgb, ref_T = [], []
    for cam in cams:
        r = torch.empty((3, cam.H, cam.W), device="cuda")
        t = torch.empty((cam.H, cam.W), device="cuda")
        ctx.gs_render(st, camera(cam), cam.W, cam.H, o, r, t)
        ref_rgb.append(r.cpu().numpy())
        ref_T.append(t.cpu().numpy())
    for g in (2, 9):
        ctx.gs_set_view_group(g, True)
        r = torch.full((9, 3, 144, 256), float("nan"), device="cuda")
        t = torch.full((9, 144, 256), float("nan"), device="cuda")
        ctx.gs_render_views(st, [camera(c) for c in cams], 256, 144, o, r, t)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), np.stack(ref_rgb)), g
        assert np.array_equal(t.cpu().numpy(), np.stack(ref_T)), g
    ctx.close()


@pytest.mark.parametrize("case", ["C2", "dense", "ragged"])
def test_mma_blend_is_bit_identical_across_batch_sizes(case):
    """SURVEY N2 / reading R-18: the batch size b is performance-only. The mma.sync
    blend computes every exponent with the same MMA sum whatever b, so frames are
    bit-identical for b in {32, 64, 128, 256}."""
    import torch
    from paper_2604_02120_b200 import camera, opts, scene_to_device
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    st = scene_to_device(scene)
    outs = []
    for b in (32, 64, 128, 256):
        r = torch.full((3, cam.H, cam.W), float("nan"), device="cuda")
        t = torch.full((cam.H, cam.W), float("nan"), device="cuda")
        ctx.gs_render(st, camera(cam), cam.W, cam.H,
                      opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_MMA, flags=1, batch=b), r, t)
        outs.append((r.cpu().numpy(), t.cpu().numpy()))
    for r, t in outs[1:]:
        assert np.array_equal(r, outs[0][0]) and np.array_equal(t, outs[0][1])
    with pytest.raises(GsError):
        ctx.gs_render(st, camera(cam), cam.W, cam.H, opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_MMA,
                                                          batch=48), r, t)


# ---- GS_FLAG_OBOX: the opacity-aware box (docs/preprocess_order.md 10b) ----
@pytest.mark.parametrize("case", list(CASES))
def test_obox_preprocess_and_binning_bit_exact(case):
    """With GS_FLAG_OBOX the rects, tiles_touched, sorted keys, values and tile ranges
    are bit-exact against the oracle's step-10b preprocess and plain-definition binning."""
    from paper_2604_02120_b200 import GS_FLAG_OBOX
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    got = gpu_preprocess(ctx, scene, cam, flags=GS_FLAG_OBOX)
    pre = oracle.preprocess(scene, cam, obox=True)
    vis = pre["touched"] > 0
    assert np.array_equal(got["touched"], pre["touched"])
    assert np.array_equal(got["rect"][vis], pre["rect"][vis])
    code, K, b = gpu_binning(ctx, scene, cam, flags=GS_FLAG_OBOX)
    assert code == 0
    ref = oracle.binning(pre, cam.W, cam.H)
    assert K == ref["K"]
    assert np.array_equal(b["keys"], ref["keys"])
    assert np.array_equal(b["vals"], ref["vals"])
    assert np.array_equal(b["ranges"], ref["ranges"])


@pytest.mark.parametrize("case", list(CASES))
def test_obox_renders_bit_identical(case):
    """Dropped pairs are alpha-skipped anyway: the frame equals the vanilla-rect one."""
    from paper_2604_02120_b200 import GS_FLAG_OBOX
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    a, ta = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC)
    b, tb = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, flags=GS_FLAG_OBOX)
    assert np.array_equal(a, b) and np.array_equal(ta, tb)


def test_stream_wait_group_orders_frame_consumers():
    """gs_stream_wait_group(stream, g): a side stream that waits for view group g sees
    the finished frames of that group (the multi-GPU gather consumes frames this way);
    groups outside the last call are rejected."""
    import torch
    from paper_2604_02120_b200 import Context, camera, opts, scene_to_device
    scene = synth.unbounded_scene(40000, 109, sh_degree=3)
    cams = synth.orbit_cameras(7, 256, 160, 1.0)
    ctx = Context(0, max_points=scene.n, max_keys=1 << 22, max_w=256, max_h=160)
    ctx.gs_set_view_group(3, True)
    st = scene_to_device(scene)
    o = opts((0.0, 0.0, 0.0), sh_degree=3)
    r = torch.full((7, 3, 160, 256), float("nan"), device="cuda")
    t = torch.full((7, 160, 256), float("nan"), device="cuda")
    side = torch.cuda.Stream()
    copies = torch.empty_like(r)
    ctx.gs_render_views(st, [camera(c) for c in cams], 256, 160, o, r, t)
    for g in range(3):
        ctx.gs_stream_wait_group(side, g)
        with torch.cuda.stream(side):
            copies[3 * g:3 * g + 3].copy_(r[3 * g:3 * g + 3])
    torch.cuda.synchronize()
    assert torch.equal(copies, r) and not torch.isnan(r).any()
    with pytest.raises(GsError):
        ctx.gs_stream_wait_group(side, 3)
    # gs_stream_wait_view: the same per view (the gather chunks of the multi-GPU orbit)
    r.fill_(float("nan"))
    copies.fill_(0.0)
    ctx.gs_render_views(st, [camera(c) for c in cams], 256, 160, o, r, t)
    for v in range(7):
        ctx.gs_stream_wait_view(side, v)
        with torch.cuda.stream(side):
            copies[v].copy_(r[v])
    torch.cuda.synchronize()
    assert torch.equal(copies, r) and not torch.isnan(r).any()
    with pytest.raises(GsError):
        ctx.gs_stream_wait_view(side, 7)
    ctx.close()


@pytest.mark.parametrize("case", ["C2", "ragged", "tall"])
@pytest.mark.parametrize("n_bands", [3, 5])
def test_row_bands_compose_the_full_frame(case, n_bands):
    """SURVEY 8(e) option, tile-row split of one view: rendering band k of n into a
    shared buffer writes only that band's rows, bit-identical to the full frame, and
    the band's binning is the oracle's lists on the band's tiles (empty elsewhere)."""
    import torch
    from paper_2604_02120_b200 import camera, opts, scene_to_device
    from paper_2604_02120_b200.orbit import band_pixel_rows
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    st = scene_to_device(scene)
    full, fT = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, st=st, flags=16)
    r = torch.full((3, cam.H, cam.W), float("nan"), device="cuda")
    t = torch.full((cam.H, cam.W), float("nan"), device="cuda")
    for k in range(n_bands):
        before = r.clone()
        ctx.gs_render(st, camera(cam), cam.W, cam.H,
                      opts(bg, sh_degree=scene.sh_degree, flags=1 | 16, band=k, n_bands=n_bands), r, t)
        torch.cuda.synchronize()
        rows = band_pixel_rows(cam.H, k, n_bands)
        other = torch.ones(cam.H, dtype=torch.bool, device="cuda")
        other[rows.start:rows.stop] = False
        assert torch.equal(r[:, other].isnan(), before[:, other].isnan())   # nothing else written
    assert np.array_equal(r.cpu().numpy().astype(np.float64), full)
    assert np.array_equal(t.cpu().numpy().astype(np.float64), fT)
    # binning of one band = the oracle's (OBOX) lists on the band's tiles
    pre = oracle.preprocess(scene, cam, obox=True)
    ref = oracle.binning(pre, cam.W, cam.H)
    gx = (cam.W + 15) // 16
    k = n_bands // 2
    code, K, b = None, None, None
    keys = torch.empty(1 << 22, dtype=torch.int64, device="cuda")
    vals = torch.empty(1 << 22, dtype=torch.int32, device="cuda")
    ranges = torch.empty((len(ref["ranges"]), 2), dtype=torch.int32, device="cuda")
    code, K = ctx.gs_debug_binning(st, camera(cam), cam.W, cam.H,
                                   opts(sh_degree=scene.sh_degree, flags=16, band=k, n_bands=n_bands),
                                   keys, vals, ranges)
    assert code == 0
    rg = ranges.cpu().numpy().view(np.uint32)
    kv = keys[:K].cpu().numpy().view(np.uint64)
    vv = vals[:K].cpu().numpy().view(np.uint32)
    gy = (cam.H + 15) // 16
    y0, y1 = k * gy // n_bands, (k + 1) * gy // n_bands
    for tile in range(len(rg)):
        a0, a1 = ref["ranges"][tile]
        if y0 <= tile // gx < y1:
            g0, g1 = rg[tile]
            assert np.array_equal(vv[g0:g1], ref["vals"][a0:a1]) and np.array_equal(kv[g0:g1], ref["keys"][a0:a1])
        else:
            assert rg[tile, 1] == rg[tile, 0]


def test_obox_opacity_edge_cases_bit_exact():
    """Step 10b at its edges: 255*o just below / at / above 1 (cull boundary), o -> 1,
    huge and tiny splats; rects and culls bit-exact against the oracle."""
    from paper_2604_02120_b200 import GS_FLAG_OBOX
    scene = synth.object_scene(4096, 110, sh_degree=1)
    edge = np.array([np.nextafter(np.float32(1 / 255), np.float32(0)), np.float32(1 / 255),
                     np.nextafter(np.float32(1 / 255), np.float32(1)), np.float32(0.004), np.float32(0.99999),
                     np.float32(1.0), np.float32(0.5), np.float32(1e-6)], np.float32)
    scene.opacity[:] = edge[np.arange(scene.n) % len(edge)]
    scene.scales[::7] *= 40.0
    scene.scales[3::7] *= 0.01
    cam = synth.look_at((0.3, -0.4, -3.0), (0, 0, 0), 200, 136, 0.9)
    ctx = make_ctx(scene, cam)
    got = gpu_preprocess(ctx, scene, cam, flags=GS_FLAG_OBOX)
    pre = oracle.preprocess(scene, cam, obox=True)
    assert np.array_equal(got["touched"], pre["touched"])
    vis = pre["touched"] > 0
    assert np.array_equal(got["rect"][vis], pre["rect"][vis])
    t = np.float32(255.0) * scene.opacity.astype(np.float32)   # the binary32 product step 10b tests
    assert not vis[t < 1.0].any()
    assert vis[t >= 1.0].any()


def test_host_async_entry_point_matches_device_frames():
    """gs_render_views_host_async back to back (double-buffered scene staging, frames
    copied back on a side stream) gives the frames of gs_render_views, call after call."""
    import torch
    from paper_2604_02120_b200 import Context, camera, opts, scene_to_device, scene_to_host
    scene = synth.unbounded_scene(30000, 111, sh_degree=3)
    cams = synth.orbit_cameras(9, 192, 128, 1.0)
    ctx = Context(0, max_points=scene.n, max_keys=1 << 22, max_w=192, max_h=128)
    ctx.gs_set_view_group(4, True)
    o = opts((0.2, 0.1, 0.0), sh_degree=3, flags=16)
    st = scene_to_device(scene)
    r = torch.empty((9, 3, 128, 192), device="cuda")
    t = torch.empty((9, 128, 192), device="cuda")
    ctx.gs_render_views(st, [camera(c) for c in cams], 192, 128, o, r, t)
    torch.cuda.synchronize()
    ref_r, ref_t = r.cpu(), t.cpu()
    hs = scene_to_host(scene)
    outs = [(torch.full((9, 3, 128, 192), float("nan")).pin_memory(), torch.full((9, 128, 192), float("nan")).pin_memory())
            for _ in range(3)]
    for hr, ht in outs:   # three calls in flight on one stream
        ctx.gs_render_views_host(hs, [camera(c) for c in cams], 192, 128, o, hr, ht, async_=True)
    torch.cuda.synchronize()
    for hr, ht in outs:
        assert torch.equal(hr, ref_r) and torch.equal(ht, ref_t)
    ctx.close()


def test_capacity_error_in_any_view_of_an_orbit_is_reported():
    """A multi-view call fails with GS_ERR_CAPACITY if any view overflows max_keys (the
    views reuse their counters, so the error is accumulated per call), and reports the
    largest K; an empty scene renders background through the orbit path."""
    import torch
    from paper_2604_02120_b200 import Context, camera, opts, scene_to_device
    scene = synth.unbounded_scene(20000, 112, sh_degree=1)
    cams = synth.orbit_cameras(6, 160, 96, 1.0)
    ks = []
    for c in cams:   # K of each view, one at a time
        ctx1 = Context(0, max_points=scene.n, max_keys=1 << 22, max_w=160, max_h=96)
        _, K, _ = gpu_binning(ctx1, scene, c)
        ks.append(K)
    cap = sorted(ks)[-2]   # only the largest view overflows
    assert cap < max(ks)
    ctx = Context(0, max_points=scene.n, max_keys=cap, max_w=160, max_h=96)
    ctx.gs_set_view_group(4, True)
    st = scene_to_device(scene)
    r = torch.empty((6, 3, 96, 160), device="cuda")
    t = torch.empty((6, 96, 160), device="cuda")
    order = sorted(range(6), key=lambda v: ks[v])        # the overflowing view is rendered first
    cam_list = [camera(cams[v]) for v in reversed(order)]
    with pytest.raises(GsError) as e:
        ctx.gs_render_views(st, cam_list, 160, 96, opts(sh_degree=1, flags=1), r, t)
    assert e.value.code == -3
    assert ctx.gs_last_stats().n_keys == max(ks)
    empty = synth.object_scene(0, 0, sh_degree=0)
    ctx0 = Context(0, max_points=1, max_keys=1024, max_w=40, max_h=24)
    r0 = torch.empty((3, 3, 24, 40), device="cuda")
    t0 = torch.empty((3, 24, 40), device="cuda")
    ctx0.gs_render_views(scene_to_device(empty), [camera(c) for c in synth.orbit_cameras(3, 40, 24, 1.0)], 40, 24,
                         opts((0.1, 0.2, 0.3), sh_degree=0, flags=1), r0, t0)
    torch.cuda.synchronize()
    assert (t0 == 1.0).all() and (r0[:, 2] == np.float32(0.3)).all()


@pytest.mark.parametrize("seed", [201, 202, 203, 204, 205, 206])
def test_random_scenes_and_cameras_bit_exact(seed):
    """Randomised coverage of the preprocess op order (FMA / reciprocal form) and the
    binning: random mixes of object and unbounded scenes, random scale spreads (tiny to
    huge), random orbit cameras and resolutions, both intersection modes; preprocess
    outputs and keys / values / ranges bit-exact, frame within the bar."""
    rng = np.random.default_rng(seed)
    from paper_2604_02120_b200 import GS_FLAG_OBOX
    n = int(rng.integers(500, 6000))
    scene = (synth.object_scene if seed % 2 else synth.unbounded_scene)(n, seed, sh_degree=int(rng.integers(0, 4)))
    scene.scales *= np.exp(rng.normal(0.0, 1.5, scene.scales.shape)).astype(np.float32)
    W, H = int(rng.integers(17, 300)), int(rng.integers(9, 200))
    cams = synth.orbit_cameras(8, W, H, float(rng.uniform(0.4, 1.6)), radius=float(rng.uniform(2.0, 6.0)),
                               elev_deg=float(rng.uniform(-40.0, 60.0)))
    cam = cams[int(rng.integers(0, 8))]
    bg = rng.uniform(0, 1, 3).astype(np.float32)
    for obox in (False, True):
        flags = GS_FLAG_OBOX if obox else 0
        ctx = make_ctx(scene, cam)
        got = gpu_preprocess(ctx, scene, cam, flags=flags)
        pre = oracle.preprocess(scene, cam, obox=obox)
        vis = pre["touched"] > 0
        assert np.array_equal(got["touched"], pre["touched"])
        for k in BIT_EXACT_KEYS:
            a = got[k].view(np.uint32) if got[k].dtype == np.float32 else got[k].astype(np.int64)
            b = pre[k].view(np.uint32) if pre[k].dtype == np.float32 else pre[k].astype(np.int64)
            assert np.array_equal(a[vis], b[vis]), k
        code, K, gb = gpu_binning(ctx, scene, cam, flags=flags)
        assert code == 0
        ref_b = oracle.binning(pre, cam.W, cam.H)
        assert K == ref_b["K"]
        assert np.array_equal(gb["keys"], ref_b["keys"]) and np.array_equal(gb["vals"], ref_b["vals"])
        assert np.array_equal(gb["ranges"], ref_b["ranges"])
    rgb, T = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, flags=GS_FLAG_OBOX)
    _, _, ref = oracle.render(scene, cam, bg)
    check_frame(f"random/{seed}", rgb, T, ref)


def test_wide_depth_range_takes_the_fourth_pass():
    """Depths beyond znear * 2^16 (13107 at znear 0.2) make the near-plane-relative
    depth keys wider than 27 bits: the 4th radix pass and the copy back must run and the
    keys / values / ranges stay bit-exact against the oracle (huge splats far away)."""
    rng = np.random.default_rng(114)
    scene = synth.object_scene(3000, 114, sh_degree=1)
    far = rng.uniform(0.0, 1.0, scene.n) < 0.5
    scene.means[far] *= np.float32(4000.0)            # far away: depths up to ~1e4 .. 4e4
    scene.means[far, 2] += np.float32(30000.0)
    scene.scales[far] *= np.float32(3000.0)            # still a few pixels wide on screen
    cam = synth.look_at((0.0, 0.0, -4.0), (0, 0, 0), 128, 96, 0.9)
    ctx = make_ctx(scene, cam)
    pre = oracle.preprocess(scene, cam)
    assert (pre["depth"][pre["touched"] > 0] > 0.2 * 65536).any()   # the wide case is exercised
    code, K, gb = gpu_binning(ctx, scene, cam)
    assert code == 0
    ref = oracle.binning(pre, cam.W, cam.H)
    assert K == ref["K"]
    assert np.array_equal(gb["keys"], ref["keys"]) and np.array_equal(gb["vals"], ref["vals"])
    assert np.array_equal(gb["ranges"], ref["ranges"])


@pytest.mark.parametrize("variant", ["scale_0.6", "scale_1.7", "stride16_deg1", "stride9_deg0", "plain_rgb"])
def test_scale_modifier_sh_stride_and_plain_colours(variant):
    """gs_opts.scale_modifier (step 4: g_k = sm * s_k), an SH record longer than the
    evaluated degree (sh_stride > (D+1)^2: degree 1 or 0 of a degree-3 / degree-2
    record) and plain colours (sh_degree -1, shs [N,3]): preprocess outputs and
    keys / values / ranges bit-exact, frame within the bar, both intersection modes."""
    from paper_2604_02120_b200 import GS_FLAG_OBOX
    scene = synth.object_scene(4000, 301, sh_degree=3)
    cam = synth.look_at((0.4, -0.6, -3.3), (0, 0, 0), 133, 71, 0.9)
    bg = np.array([0.3, 0.1, 0.6], np.float32)
    sm = 1.0
    if variant.startswith("scale_"):
        sm = float(variant.split("_")[1])
    elif variant == "stride16_deg1":
        scene.sh_degree = 1
    elif variant == "stride9_deg0":
        scene = synth.object_scene(4000, 302, sh_degree=2)
        scene.sh_degree = 0
    else:
        scene.shs = np.ascontiguousarray(np.clip(scene.shs[:, 0, :] * 0.28 + 0.5, 0.0, 1.0), np.float32)
        scene.sh_degree = -1
    for obox in (False, True):
        flags = GS_FLAG_OBOX if obox else 0
        ctx = make_ctx(scene, cam)
        got = gpu_preprocess(ctx, scene, cam, flags=flags, scale_modifier=sm)
        pre = oracle.preprocess(scene, cam, scale_modifier=sm, obox=obox)
        assert pre["n_visible"] > 1000
        vis = pre["touched"] > 0
        assert np.array_equal(got["touched"], pre["touched"])
        for k in BIT_EXACT_KEYS:
            a = got[k].view(np.uint32) if got[k].dtype == np.float32 else got[k].astype(np.int64)
            b = pre[k].view(np.uint32) if pre[k].dtype == np.float32 else pre[k].astype(np.int64)
            assert np.array_equal(a[vis], b[vis]), k
        code, K, gb = gpu_binning(ctx, scene, cam, flags=flags, scale_modifier=sm)
        assert code == 0
        ref_b = oracle.binning(pre, cam.W, cam.H)
        assert K == ref_b["K"] and np.array_equal(gb["keys"], ref_b["keys"])
        assert np.array_equal(gb["vals"], ref_b["vals"]) and np.array_equal(gb["ranges"], ref_b["ranges"])
        rgb, T = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, flags=flags, scale_modifier=sm)
        _, _, ref = oracle.render(scene, cam, bg, obox=obox, scale_modifier=sm)
        check_frame(f"inputs/{variant}/{'obox' if obox else 'vanilla'}", rgb, T, ref)


@pytest.mark.parametrize("obox", [False, True], ids=["vanilla", "obox"])
def test_capacity_boundary_is_exact(obox):
    """max_keys == K renders (keys / values / ranges bit-exact, frame within the bar);
    max_keys == K - 1 is a capacity error that reports the exact K, for gs_render and
    for a view group (gs_render_views)."""
    import torch
    from paper_2604_02120_b200 import GS_FLAG_OBOX, camera, opts, scene_to_device
    scene, cams, bg = synth.make_config("C2", n_override=60000, views=3)
    cam = cams[0]
    flags = GS_FLAG_OBOX if obox else 0
    pre = oracle.preprocess(scene, cam, obox=obox)
    K = oracle.binning(pre, cam.W, cam.H)["K"]
    st = scene_to_device(scene)
    ctx = make_ctx(scene, cam, max_keys=K)
    code, Kg, gb = gpu_binning(ctx, scene, cam, capacity=K, st=st, flags=flags)
    assert code == 0 and Kg == K
    ref_b = oracle.binning(pre, cam.W, cam.H)
    assert np.array_equal(gb["keys"], ref_b["keys"]) and np.array_equal(gb["vals"], ref_b["vals"])
    rgb, T = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, st=st, flags=flags)
    _, _, ref = oracle.render(scene, cam, bg, obox=obox)
    check_frame(f"capacity_boundary/{'obox' if obox else 'vanilla'}", rgb, T, ref)
    ctx.close()
    ctx = make_ctx(scene, cam, max_keys=K - 1)
    with pytest.raises(GsError) as e:
        gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, st=st, flags=flags)
    assert e.value.code == -3 and ctx.gs_last_stats().n_keys == K
    # the same view inside a group of 3: only its K exceeds the capacity when it is the largest
    Ks = [oracle.binning(oracle.preprocess(scene, c, obox=obox), c.W, c.H)["K"] for c in cams]
    ctx.close()
    ctx = make_ctx(scene, cam, max_keys=max(Ks))
    ctx.gs_set_view_group(3, True)
    grgb = torch.empty((3, 3, cam.H, cam.W), device="cuda")
    gT = torch.empty((3, cam.H, cam.W), device="cuda")
    o = opts(bg, sh_degree=scene.sh_degree, flags=1 | flags)
    ctx.gs_render_views(st, [camera(c) for c in cams], cam.W, cam.H, o, grgb, gT)
    torch.cuda.synchronize()
    ctx.close()
    ctx = make_ctx(scene, cam, max_keys=max(Ks) - 1)
    ctx.gs_set_view_group(3, True)
    with pytest.raises(GsError) as e:
        ctx.gs_render_views(st, [camera(c) for c in cams], cam.W, cam.H, o, grgb, gT)
        torch.cuda.synchronize()
    assert e.value.code == -3 and ctx.gs_last_stats().n_keys == max(Ks)
    ctx.close()


@pytest.mark.parametrize("wh", [(1, 1), (16, 16), (17, 1), (1, 33)], ids=["1x1", "16x16", "17x1", "1x33"])
@pytest.mark.parametrize("n", [1, 2, 300])
def test_degenerate_image_and_scene_sizes(wh, n):
    """One-pixel and one-tile images, one-row / one-column images with a ragged tile,
    one or two Gaussians: preprocess / binning bit-exact, frame within the bar."""
    W, H = wh
    scene = synth.object_scene(n, 400 + n, sh_degree=3)
    if n <= 2:
        scene.means[:] = np.array([[0.0, 0.0, 0.0], [0.05, -0.02, 0.3]], np.float32)[:n]
        scene.scales[:] = 0.4
        scene.opacity[:] = 0.8
    cam = synth.look_at((0.0, 0.0, -3.0), (0, 0, 0), W, H, 0.9)
    bg = np.array([0.25, 0.5, 0.75], np.float32)
    for obox in (False, True):
        from paper_2604_02120_b200 import GS_FLAG_OBOX
        flags = GS_FLAG_OBOX if obox else 0
        ctx = make_ctx(scene, cam)
        got = gpu_preprocess(ctx, scene, cam, flags=flags)
        pre = oracle.preprocess(scene, cam, obox=obox)
        vis = pre["touched"] > 0
        if n <= 2:
            assert vis.all()
        assert np.array_equal(got["touched"], pre["touched"])
        for k in BIT_EXACT_KEYS:
            a = got[k].view(np.uint32) if got[k].dtype == np.float32 else got[k].astype(np.int64)
            b = pre[k].view(np.uint32) if pre[k].dtype == np.float32 else pre[k].astype(np.int64)
            assert np.array_equal(a[vis], b[vis]), k
        code, K, gb = gpu_binning(ctx, scene, cam, flags=flags)
        ref_b = oracle.binning(pre, W, H)
        assert code == 0 and K == ref_b["K"]
        if K:
            assert np.array_equal(gb["keys"], ref_b["keys"]) and np.array_equal(gb["vals"], ref_b["vals"])
        assert np.array_equal(gb["ranges"], ref_b["ranges"])
        for blend in (GS_BLEND_TC, GS_BLEND_DIRECT, GS_BLEND_MMA):
            rgb, T = gpu_render(ctx, scene, cam, bg, blend, flags=flags)
            _, _, ref = oracle.render(scene, cam, bg, obox=obox)
            check_frame(f"degenerate/{W}x{H}/n{n}/{'obox' if obox else 'vanilla'}/{['tc', 'direct', 'mma', 'tc_color'][blend]}",
                        rgb, T, ref)


def test_single_view_calls_interleaved_with_static_scene_view_groups():
    """gs_render (the context's own workspace, caller's stream) enqueued back to back with
    gs_render_views under GS_FLAG_STATIC_SCENE (whose preprocess does not wait for the
    caller's earlier work): the two share no buffer, so every frame equals its reference."""
    import torch
    from paper_2604_02120_b200 import GS_FLAG_STATIC_SCENE, Context, camera, opts, scene_to_device
    scene = synth.unbounded_scene(200000, 115, sh_degree=3)
    cams = synth.orbit_cameras(6, 640, 360, 1.0)
    ctx = Context(0, max_points=scene.n, max_keys=1 << 23, max_w=640, max_h=360)
    ctx.gs_set_view_group(4, True)
    st = scene_to_device(scene)
    o = opts((0.1, 0.2, 0.3), sh_degree=3)
    ref_r, ref_t = [], []
    for c in cams:
        r = torch.empty((3, 360, 640), device="cuda")
        t = torch.empty((360, 640), device="cuda")
        ctx.gs_render(st, camera(c), 640, 360, o, r, t)
        torch.cuda.synchronize()
        ref_r.append(r.cpu())
        ref_t.append(t.cpu())
    o_s = opts((0.1, 0.2, 0.3), sh_degree=3, flags=GS_FLAG_STATIC_SCENE)
    outs = []
    for it in range(3):
        r1 = torch.full((3, 360, 640), float("nan"), device="cuda")
        t1 = torch.full((360, 640), float("nan"), device="cuda")
        rv = torch.full((5, 3, 360, 640), float("nan"), device="cuda")
        tv = torch.full((5, 360, 640), float("nan"), device="cuda")
        ctx.gs_render(st, camera(cams[0]), 640, 360, o, r1, t1)
        ctx.gs_render_views(st, [camera(c) for c in cams[1:]], 640, 360, o_s, rv, tv)
        outs.append((r1, t1, rv, tv))
    torch.cuda.synchronize()
    for r1, t1, rv, tv in outs:
        assert torch.equal(r1.cpu(), ref_r[0]) and torch.equal(t1.cpu(), ref_t[0])
        for v in range(5):
            assert torch.equal(rv[v].cpu(), ref_r[v + 1]) and torch.equal(tv[v].cpu(), ref_t[v + 1])
    ctx.close()


def test_workspace_allocation_failure_leaves_the_context_usable():
    """A view group whose per-view workspaces do not fit in HBM fails with GS_ERR_CUDA
    (no crash, nothing half-allocated); the context then still renders correct frames."""
    import torch
    from paper_2604_02120_b200 import GS_ERR_CUDA, Context, camera, opts, scene_to_device
    scene = synth.object_scene(20000, 116, sh_degree=1)
    cams = synth.orbit_cameras(3, 160, 96, 1.0)
    free, _ = torch.cuda.mem_get_info()
    # a max_keys whose workspace (16 B per key) takes about a fifth of the free memory:
    # 16 views x 2 slot sets cannot all be allocated
    max_keys = min((1 << 32) - 1, int(free * 0.2 / 17))
    ctx = Context(0, max_points=scene.n, max_keys=max_keys, max_w=160, max_h=96)
    st = scene_to_device(scene)
    o = opts((0.0, 0.0, 0.0), sh_degree=1)
    ref = []
    for c in cams:
        r = torch.empty((3, 96, 160), device="cuda")
        t = torch.empty((96, 160), device="cuda")
        ctx.gs_render(st, camera(c), 160, 96, o, r, t)
        ref.append(r.cpu())
    ctx.gs_set_view_group(16, True)
    rv = torch.empty((3 * 8, 3, 96, 160), device="cuda")
    tv = torch.empty((3 * 8, 96, 160), device="cuda")
    with pytest.raises(GsError) as e:
        ctx.gs_render_views(st, [camera(c) for c in cams] * 8, 160, 96, o, rv, tv)
    assert e.value.code == GS_ERR_CUDA
    torch.cuda.synchronize()
    ctx.gs_set_view_group(2, False)        # the slots of set 0 that did get allocated
    rv.fill_(float("nan"))
    ctx.gs_render_views(st, [camera(c) for c in cams], 160, 96, o, rv[:3], tv[:3])
    torch.cuda.synchronize()
    for v in range(3):
        assert torch.equal(rv[v].cpu(), ref[v])
    r = torch.empty((3, 96, 160), device="cuda")
    t = torch.empty((96, 160), device="cuda")
    ctx.gs_render(st, camera(cams[1]), 160, 96, o, r, t)
    torch.cuda.synchronize()
    assert torch.equal(r.cpu(), ref[1])
    ctx.close()


@pytest.mark.parametrize("case", ["C2", "dense", "ragged", "adversarial"])
def test_supertile_and_per_tile_lists_render_identically(case):
    """GS_FLAG_TILE_LISTS bins into per-tile lists for the tcgen05 blend (the lists the other
    blends read); the default supertile lists, filtered by the blend's producer, hold the
    same per-tile sequences, so the frames are bit-identical."""
    from paper_2604_02120_b200 import GS_FLAG_OBOX, GS_FLAG_TILE_LISTS
    scene, cam, bg = CASES[case]()
    ctx = make_ctx(scene, cam)
    for flags in (0, GS_FLAG_OBOX):
        a, ta = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, flags=flags)
        b, tb = gpu_render(ctx, scene, cam, bg, GS_BLEND_TC, flags=flags | GS_FLAG_TILE_LISTS)
        assert np.array_equal(a, b) and np.array_equal(ta, tb)
