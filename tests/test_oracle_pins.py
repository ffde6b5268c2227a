"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test checks the oracle against something other than itself: worked
examples printed in SPEC.md (tests/golden/), closed forms, invariants,
textbook/library routines (scipy rotations, finite differences, quadrature
orthonormality of the SH basis) and brute force on tiny inputs.
P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2604_02120_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _scene(means, scales, rots, opac, shs, deg):
    return synth.Scene(np.asarray(means, np.float32).reshape(-1, 3),
                       np.asarray(scales, np.float32).reshape(-1, 3),
                       np.asarray(rots, np.float32).reshape(-1, 4),
                       np.asarray(opac, np.float32).reshape(-1),
                       np.asarray(shs, np.float32), deg)


def _axis_camera(W=64, H=64, f=50.0, D=10.0, campos=(0.0, 0.0, -10.0)):
    """Identity-rotation camera at (0,0,-D): world point (0,0,0) at depth D."""
    return synth.Camera(R=np.eye(3, dtype=np.float32), t=np.array([0, 0, D], np.float32),
                        fx=f, fy=f, cx=(W - 1) / 2, cy=(H - 1) / 2, znear=0.2,
                        tan_fovx=float(np.float32(W / (2 * f))),
                        tan_fovy=float(np.float32(H / (2 * f))),
                        campos=np.array(campos, np.float32), W=W, H=H)


# --------------------------------------------------------------------------
# Eq. (3) == Eq. (6): the GEMM-compatible rewrite
# --------------------------------------------------------------------------

def test_eq6_worked_examples_from_spec():
    g = json.load(open(os.path.join(GOLD, "eq6_worked_example.json")))
    for c in g["v_g"]:
        np.testing.assert_array_equal(oracle.vg(*c["conic"], *c["xhat"]), c["v"])
    for c in g["v_p"]:
        np.testing.assert_array_equal(oracle.vp(*c["xbar"]), c["v"])
    assert float(np.dot(g["dot"]["v_g"], g["dot"]["v_p"])) == g["dot"]["value"]
    # power_ref examples through the Eq. (6) path, with xbar = 0 (pixel = reference)
    for c in g["power_ref"]:
        A, B, C = c["conic"]
        dx, dy = c["delta"]
        assert float(oracle.vg(A, B, C, dx, dy) @ oracle.vp(0, 0)) == c["power"]


def test_eq6_identity_random_and_sign_convention():
    """power(x_g - x_p) == v_g(x_g - x_c) . v_p(x_c - x_p)  (Eq. 4-6).

    A mirrored convention (x_bar = x_p - x_c, as SPEC S:311/S:330 would read)
    fails this test: see test_mirrored_convention_fails."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        L = rng.normal(size=(2, 2))
        Sinv = L @ L.T + 0.1 * np.eye(2)
        A, B, C = Sinv[0, 0], Sinv[0, 1], Sinv[1, 1]
        xg, yg = rng.uniform(-50, 50, 2)
        xc, yc = 7.5, 7.5
        xp, yp = rng.integers(0, 16, 2)
        dx, dy = xg - xp, yg - yp
        direct = -0.5 * A * dx * dx - B * dx * dy - 0.5 * C * dy * dy
        gemm = oracle.vg(A, B, C, xg - xc, yg - yc) @ oracle.vp(xc - xp, yc - yp)
        assert abs(gemm - direct) <= 1e-9 * (1 + abs(direct))


def test_mirrored_convention_fails():
    A, B, C = 2.0, 1.0, 3.0
    xg, yg, xc, yc, xp, yp = 1.0, 2.0, 7.5, 7.5, 3.0, 12.0
    dx, dy = xg - xp, yg - yp
    direct = -0.5 * A * dx * dx - B * dx * dy - 0.5 * C * dy * dy
    mirrored = oracle.vg(A, B, C, xg - xc, yg - yc) @ oracle.vp(xp - xc, yp - yc)
    assert abs(mirrored - direct) > 1.0


def test_pixel_matrix_row_sums_closed_form():
    """Centre reference (7.5, 7.5): sum xb = sum yb = sum xb*yb = 0,
    sum xb^2 = sum yb^2 = 16 * sum_k (k-7.5)^2 = 16*340 = 5440, sum 1 = 256."""
    cols = np.array([oracle.vp(7.5 - x, 7.5 - y) for y in range(16) for x in range(16)])
    s = cols.sum(0)
    np.testing.assert_array_equal(s, [5440.0, 5440.0, 0.0, 0.0, 0.0, 256.0])
    assert sum((k - 7.5) ** 2 for k in range(16)) == 340.0


# --------------------------------------------------------------------------
# Preprocess (formulas per docs/preprocess_order.md)
# --------------------------------------------------------------------------

def _sh_zero(n, deg):
    return np.zeros((n, (deg + 1) ** 2, 3), np.float32)


def test_sh_constant_cases():
    """zero coeffs -> 0.5; DC only -> C0*k + 0.5; negative -> 0."""
    n = 3
    means = np.zeros((n, 3)); means[:, 0] = [-0.1, 0.0, 0.1]
    shs = _sh_zero(n, 3)
    shs[1, 0, :] = [0.7, -0.3, 1.1]
    shs[2, 0, :] = [-5.0, -5.0, -5.0]
    sc = _scene(means, np.full((n, 3), 0.05), np.tile([1, 0, 0, 0], (n, 1)), np.full(n, 0.5), shs, 3)
    pre = oracle.preprocess(sc, _axis_camera())
    assert (pre["touched"] > 0).all()
    np.testing.assert_array_equal(pre["rgb"][0], [0.5, 0.5, 0.5])
    C0 = np.float32(0.28209479177387814)
    exp1 = np.maximum(C0 * shs[1, 0] + np.float32(0.5), 0).astype(np.float32)
    np.testing.assert_array_equal(pre["rgb"][1], exp1)
    np.testing.assert_array_equal(pre["rgb"][2], [0.0, 0.0, 0.0])


def test_sh_basis_orthonormal_by_quadrature():
    """The 16 real SH basis functions used by the colour stage are orthonormal
    on the sphere (Gram error small), which fails for a wrong constant, sign-
    insensitive but polynomial-typo-sensitive; plus degree check against
    scipy's complex spherical harmonics."""
    from scipy.special import sph_harm_y
    nt, nphi = 10, 24
    xs, ws = np.polynomial.legendre.leggauss(nt)          # cos(theta) nodes
    dirs, wq = [], []
    for ct, w in zip(xs, ws):
        st = math.sqrt(1 - ct * ct)
        for k in range(nphi):
            ph = 2 * math.pi * k / nphi
            dirs.append((st * math.cos(ph), st * math.sin(ph), ct))
            wq.append(w * 2 * math.pi / nphi)
    dirs = np.array(dirs); wq = np.array(wq)
    n = len(dirs)
    # Gaussians on a unit sphere around campos = origin, seen from far away
    cam = _axis_camera(W=64, H=64, f=1000.0, D=1000.0, campos=(0, 0, 0))
    Y = np.zeros((16, n))
    for k in range(16):
        shs = _sh_zero(n, 3)
        shs[:, k, 0] = 0.1
        sc = _scene(dirs, np.full((n, 3), 0.01), np.tile([1, 0, 0, 0], (n, 1)), np.full(n, 0.5), shs, 3)
        pre = oracle.preprocess(sc, cam)
        assert (pre["touched"] > 0).all()
        base = np.float32(0.5) if k else None
        val = pre["rgb"][:, 0].astype(np.float64)
        if k == 0:
            Y[k] = (val - 0.5) / 0.1
        else:
            # res = C0*0 + ... = 0.1*Y_k; rgb = res + 0.5
            Y[k] = (val - float(base)) / 0.1
    G = (Y * wq) @ Y.T
    assert np.abs(G - np.eye(16)).max() < 2e-5, np.abs(G - np.eye(16)).max()
    # degree l functions live in span of complex Y_l^m
    theta = np.arccos(dirs[:, 2]); phi = np.arctan2(dirs[:, 1], dirs[:, 0])
    for l in range(4):
        Z = np.array([sph_harm_y(l, m, theta, phi) for m in range(-l, l + 1)])
        for k in range(l * l, (l + 1) ** 2):
            proj = (Z.conj() * wq) @ Y[k]
            assert abs(np.sum(np.abs(proj) ** 2) - 1.0) < 5e-5


def test_projection_on_axis_isotropic_closed_form():
    """on-axis isotropic Gaussian -> cov2D = (f s / z)^2 + 0.3, B = 0;
    radius r = ceil(3 sqrt(a + sqrt(0.1))) (lambda floor)."""
    f, z, s = 50.0, 10.0, 0.05
    sc = _scene([[0, 0, 0]], [[s, s, s]], [[1, 0, 0, 0]], [0.5], _sh_zero(1, 0), 0)
    pre = oracle.preprocess(sc, _axis_camera(f=f, D=z))
    a = (f * s / z) ** 2 + 0.3
    A, B, C = pre["conic"][0]
    assert B == 0.0
    assert abs(1 / A - a) < 1e-5 * a and abs(1 / C - a) < 1e-5 * a
    assert pre["radius"][0] == math.ceil(3 * math.sqrt(a + math.sqrt(0.1)))
    assert pre["depth"][0] == np.float32(z)
    np.testing.assert_allclose(pre["xy"][0], [31.5, 31.5])


def test_projection_matches_finite_difference_jacobian():
    """cov2D - 0.3 I == J Sigma J^T with J the finite-difference Jacobian of the
    pinhole projection (textbook EWA), Sigma = R(q) diag(s^2) R(q)^T from scipy."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(3)
    n = 200
    means = rng.uniform(-1.5, 1.5, (n, 3)); means[:, 2] = rng.uniform(-2, 2, n)
    scales = np.exp(rng.uniform(np.log(0.01), np.log(0.2), (n, 3)))
    q = rng.normal(size=(n, 4)); q /= np.linalg.norm(q, axis=1, keepdims=True)
    cam = synth.look_at((0.3, -0.5, -6.0), (0, 0, 0), 320, 240, 0.9)
    sc = _scene(means, scales, q, np.full(n, 0.5), _sh_zero(n, 0), 0)
    pre = oracle.preprocess(sc, cam)
    R = cam.R.astype(np.float64); t = cam.t.astype(np.float64)

    def proj(p):
        v = R @ p + t
        return np.array([cam.fx * v[0] / v[2] + cam.cx, cam.fy * v[1] / v[2] + cam.cy])

    checked = 0
    for i in range(n):
        if pre["touched"][i] == 0:
            continue
        p = means[i].astype(np.float32).astype(np.float64)
        v = R @ p + t
        if abs(v[0] / v[2]) > 1.2 * cam.tan_fovx or abs(v[1] / v[2]) > 1.2 * cam.tan_fovy:
            continue           # outside the un-clamped region
        h = 1e-4
        J = np.stack([(proj(p + h * e) - proj(p - h * e)) / (2 * h) for e in np.eye(3)], 1)
        rot = Rotation.from_quat(np.roll(q[i].astype(np.float32).astype(np.float64), -1)).as_matrix()
        s = scales[i].astype(np.float32).astype(np.float64)
        Sig = rot @ np.diag(s * s) @ rot.T
        cov = J @ Sig @ J.T
        A, B, C = pre["conic"][i].astype(np.float64)
        inv = np.linalg.inv(np.array([[A, B], [B, C]]))
        ref = cov + 0.3 * np.eye(2)
        assert np.abs(inv - ref).max() <= 2e-4 * np.abs(ref).max(), (i, inv, ref)
        np.testing.assert_allclose(pre["xy"][i], proj(p), rtol=0, atol=2e-3)
        checked += 1
    assert checked > 100


def test_rect_membership_semantics():
    """Tile column tx is in [xmin, xmax) iff 16tx+16 > mx - r and 16tx+1 <= mx + r
    (vanilla's rect, clipped to the grid; R-16). Every integer pixel within
    [mx - r, mx + r - 1] then lies in a touched tile; the pixel mx + r itself
    may not (the upper-edge off-by-one of vanilla's getRect, R-16)."""
    sc, cams, _ = synth.make_config("C1")
    cam = cams[0]
    pre = oracle.preprocess(sc, cam)
    gx = (cam.W + 15) // 16
    for i in np.nonzero(pre["touched"])[0]:
        mx = float(pre["xy"][i, 0]); r = float(pre["radius"][i])
        xmin, _, xmax, _ = pre["rect"][i]
        for tx in range(gx):
            inside = (16 * tx + 16 > mx - r) and (16 * tx + 1 <= mx + r)
            assert (xmin <= tx < xmax) == inside, (i, tx, mx, r, xmin, xmax)
        for px in range(max(0, math.ceil(mx - r)), min(cam.W, math.floor(mx + r - 1) + 1)):
            assert xmin <= px // 16 < xmax


def test_near_plane_cull_and_determinism():
    sc = _scene([[0, 0, -9.9], [0, 0, -9.7], [0, 0, 0]], np.full((3, 3), 0.05),
                np.tile([1, 0, 0, 0], (3, 1)), np.full(3, 0.5), _sh_zero(3, 0), 0)
    cam = _axis_camera(D=10.0)          # depths 0.1, 0.3, 10
    pre = oracle.preprocess(sc, cam)
    assert pre["touched"][0] == 0 and pre["touched"][1] > 0 and pre["touched"][2] > 0
    pre2 = oracle.preprocess(sc, cam)
    for k in ("depth", "xy", "conic", "rgb", "rect", "touched"):
        assert np.array_equal(pre[k], pre2[k])


# --------------------------------------------------------------------------
# Binning: brute force and invariants
# --------------------------------------------------------------------------

def _brute_binning(pre, W, H):
    gx = (W + 15) // 16
    items = []
    for i in np.nonzero(pre["touched"])[0]:
        x0, y0, x1, y1 = pre["rect"][i]
        db = int(pre["depth"][i:i + 1].view(np.uint32)[0])
        for ty in range(y0, y1):
            for tx in range(x0, x1):
                items.append((ty * gx + tx, db, int(i)))
    items.sort()
    return items


def test_binning_matches_python_sorted():
    sc, cams, _ = synth.make_config("C1")
    cam = cams[0]
    pre = oracle.preprocess(sc, cam)
    b = oracle.binning(pre, cam.W, cam.H)
    items = _brute_binning(pre, cam.W, cam.H)
    assert b["K"] == len(items) == int(pre["touched"].sum())
    keys = np.array([(t << 32) | d for t, d, _ in items], np.uint64)
    vals = np.array([i for _, _, i in items], np.uint32)
    assert np.array_equal(b["keys"], keys) and np.array_equal(b["vals"], vals)
    r = b["ranges"].astype(np.int64)
    nz = r[:, 1] > r[:, 0]
    assert r[nz, 0].min() == 0 and r[nz, 1].max() == b["K"]
    assert (r[nz][1:, 0] == r[nz][:-1, 1]).all()          # partition of [0, K)
    for t in range(len(r)):
        seg = b["keys"][r[t, 0]:r[t, 1]]
        assert ((seg >> np.uint64(32)) == t).all()
        assert (np.diff(seg.astype(np.int64)) >= 0).all()


def test_binning_equal_depth_tie_break_by_index():
    """Fronto-parallel plane: all depths equal -> ascending Gaussian index (R-12)."""
    n = 200
    rng = np.random.default_rng(5)
    means = np.zeros((n, 3)); means[:, :2] = rng.uniform(-0.5, 0.5, (n, 2))
    cam = _axis_camera(D=10.0)
    sc = _scene(means, np.full((n, 3), 0.02), np.tile([1, 0, 0, 0], (n, 1)), np.full(n, 0.5),
                _sh_zero(n, 0), 0)
    pre = oracle.preprocess(sc, cam)
    assert len(set(pre["depth"][pre["touched"] > 0].tolist())) == 1
    b = oracle.binning(pre, cam.W, cam.H)
    for t0, t1 in b["ranges"]:
        assert (np.diff(b["vals"][t0:t1].astype(np.int64)) > 0).all()


# --------------------------------------------------------------------------
# Blending (Eq. 1, Alg. 1): worked examples, closed forms, invariants
# --------------------------------------------------------------------------

def _splats(lst):
    n = len(lst)
    pre = dict(xy=np.zeros((max(n, 1), 2), np.float32), conic=np.zeros((max(n, 1), 3), np.float32),
               opacity=np.zeros(max(n, 1), np.float32), rgb=np.zeros((max(n, 1), 3), np.float32),
               touched=np.zeros(max(n, 1), np.uint32))
    for i, s in enumerate(lst):
        pre["xy"][i] = s["xy"]; pre["conic"][i] = s["conic"]; pre["opacity"][i] = s["o"]
        pre["rgb"][i] = s["rgb"]; pre["touched"][i] = 1
    return pre


def _one_tile_binning(n):
    ranges = np.zeros((1, 2), np.uint32)
    ranges[0] = (0, n) if n else (0, 0)
    return dict(vals=np.arange(max(n, 1), dtype=np.uint32), ranges=ranges, K=n)


def test_compositing_worked_examples_from_spec():
    g = json.load(open(os.path.join(GOLD, "compositing_examples.json")))
    for c in g["cases"]:
        pre = _splats(c["splats"])
        out = oracle.blend(pre, _one_tile_binning(len(c["splats"])), 16, 16, c["bg"], threads=1)
        px, py = c["pixel"]
        np.testing.assert_allclose(out["rgb"][:, py, px], c["rgb"], rtol=0, atol=1e-7)
        assert abs(out["T"][py, px] - c["T"]) < 1e-7


def test_single_isotropic_gaussian_closed_form():
    """alpha(p) = min(0.99, o exp(-|p-mu|^2 / (2 sigma^2))); out = alpha c + (1-alpha) bg
    where alpha >= 1/255, else bg; T = 1 - alpha."""
    sig2, o = 6.0, 0.8
    mu = (7.3, 8.6)
    pre = _splats([{"xy": mu, "conic": [1 / sig2, 0, 1 / sig2], "o": o, "rgb": [0.9, 0.2, 0.4]}])
    bg = np.array([0.1, 0.3, 0.5])
    out = oracle.blend(pre, _one_tile_binning(1), 16, 16, bg, threads=1)
    yy, xx = np.mgrid[0:16, 0:16]
    c32 = lambda v: float(np.float32(v))
    d2 = (xx - c32(mu[0])) ** 2 + (yy - c32(mu[1])) ** 2
    alpha = np.minimum(0.99, c32(o) * np.exp(-d2 / 2 * c32(1 / sig2)))
    keep = alpha >= np.float32(1 / 255)
    a = np.where(keep, alpha, 0.0)
    rgb = np.float32([0.9, 0.2, 0.4]).astype(np.float64)
    for ch in range(3):
        np.testing.assert_allclose(out["rgb"][ch], a * rgb[ch] + (1 - a) * bg.astype(np.float32)[ch],
                                   rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["T"], 1 - a, rtol=0, atol=1e-12)


@pytest.fixture(scope="module")
def c1():
    sc, cams, bg = synth.make_config("C1")
    cam = cams[0]
    pre = oracle.preprocess(sc, cam)
    b = oracle.binning(pre, cam.W, cam.H)
    return sc, cam, pre, b


def test_weights_plus_transmittance_is_one(c1):
    """Telescoping: sum_i w_i + T_final = 1 exactly in real arithmetic, with
    skips and early stop (Eq. 1). Colours 1, bg 0 -> out = sum w."""
    sc, cam, pre, b = c1
    p2 = dict(pre); p2["rgb"] = np.ones_like(pre["rgb"])
    out = oracle.blend(p2, b, cam.W, cam.H, (0, 0, 0), threads=2)
    assert np.abs(out["rgb"][0] + out["T"] - 1.0).max() < 1e-12
    assert (out["T"] >= 0).all() and (out["T"] <= 1).all()
    assert out["T"].min() < 1e-3          # the early-termination path is exercised


def test_zero_opacity_gives_background_exactly(c1):
    sc, cam, pre, b = c1
    p2 = dict(pre); p2["opacity"] = np.zeros_like(pre["opacity"])
    bg = (0.25, 0.5, 0.75)
    out = oracle.blend(p2, b, cam.W, cam.H, bg, threads=1)
    for ch in range(3):
        assert (out["rgb"][ch] == np.float32(bg[ch])).all()
    assert (out["T"] == 1.0).all()


def test_constant_colour_scene(c1):
    sc, cam, pre, b = c1
    p2 = dict(pre); p2["rgb"] = np.full_like(pre["rgb"], 0.375)
    out = oracle.blend(p2, b, cam.W, cam.H, (0.375, 0.375, 0.375), threads=1)
    assert np.abs(out["rgb"] - 0.375).max() < 1e-12


def test_transmittance_monotone_along_list(c1):
    """T non-increasing: truncating every tile list can only raise T."""
    sc, cam, pre, b = c1
    full = oracle.blend(pre, b, cam.W, cam.H, threads=1)
    r = b["ranges"].copy()
    r[:, 1] = np.minimum(r[:, 1], r[:, 0] + (r[:, 1] - r[:, 0]) // 2)
    b2 = dict(b); b2["ranges"] = r
    half = oracle.blend(pre, b2, cam.W, cam.H, threads=1)
    assert (half["T"] >= full["T"] - 1e-15).all()


def test_unsorted_then_sorted_brute_force(c1):
    """Per pixel: collect Gaussians whose rect holds the pixel's tile in INPUT
    order, sort by (depth, index), composite -> equals the tiled result."""
    sc, cam, pre, b = c1
    out = oracle.blend(pre, b, cam.W, cam.H, (0.1, 0.2, 0.3), threads=1)
    rng = np.random.default_rng(1)
    vis = np.nonzero(pre["touched"])[0]
    for _ in range(64):
        px, py = int(rng.integers(0, cam.W)), int(rng.integers(0, cam.H))
        tx, ty = px // 16, py // 16
        cand = [i for i in vis if pre["rect"][i, 0] <= tx < pre["rect"][i, 2]
                and pre["rect"][i, 1] <= ty < pre["rect"][i, 3]]
        cand.sort(key=lambda i: (float(pre["depth"][i]), i))
        o3, oT = oracle.blend_pixel(cand, pre, px, py, (0.1, 0.2, 0.3))
        assert np.array_equal(o3, out["rgb"][:, py, px]) and oT == out["T"][py, px]


def test_input_permutation_invariance():
    """Permuting the input Gaussians (distinct depths) leaves the image unchanged."""
    sc0, cams, bg = synth.make_config("C1")
    cam = cams[0]
    d0 = oracle.preprocess(sc0, cam)["depth"]
    _, first, cnt = np.unique(d0, return_index=True, return_counts=True)
    keep = np.sort(first[cnt == 1])                      # drop exact depth ties
    sc = synth.Scene(sc0.means[keep], sc0.scales[keep], sc0.rots[keep], sc0.opacity[keep],
                     sc0.shs[keep], sc0.sh_degree)
    perm = np.random.default_rng(2).permutation(sc.n)
    sc2 = synth.Scene(sc.means[perm], sc.scales[perm], sc.rots[perm], sc.opacity[perm],
                      sc.shs[perm], sc.sh_degree)
    _, _, o1 = oracle.render(sc, cam, bg, threads=1, mask=False)
    pre2, _, o2 = oracle.render(sc2, cam, bg, threads=1, mask=False)
    d = pre2["depth"][pre2["touched"] > 0]
    assert len(np.unique(d)) == len(d)
    assert np.array_equal(o1["rgb"], o2["rgb"]) and np.array_equal(o1["T"], o2["T"])


def test_thread_count_determinism(c1):
    sc, cam, pre, b = c1
    o1 = oracle.blend(pre, b, cam.W, cam.H, threads=1)
    o4 = oracle.blend(pre, b, cam.W, cam.H, threads=4)
    assert np.array_equal(o1["rgb"], o4["rgb"]) and np.array_equal(o1["flag"], o4["flag"])


def test_end_to_end_single_gaussian_closed_form():
    """Whole oracle path on one on-axis isotropic Gaussian: the image is the
    closed-form alpha map with sigma^2 = (f s / z)^2 + 0.3, clipped to its rect."""
    f, z, s, o = 50.0, 10.0, 0.2, 0.9
    shs = np.zeros((1, 1, 3), np.float32); shs[0, 0] = [1.0, 0.0, -1.0]
    sc = _scene([[0, 0, 0]], [[s, s, s]], [[1, 0, 0, 0]], [o], shs, 0)
    cam = _axis_camera(f=f, D=z)
    pre, b, out = oracle.render(sc, cam, (0, 0, 0), threads=1)
    sig2 = (f * s / z) ** 2 + 0.3
    yy, xx = np.mgrid[0:64, 0:64]
    d2 = (xx - 31.5) ** 2 + (yy - 31.5) ** 2
    alpha = np.minimum(0.99, np.float32(o) * np.exp(-d2 / (2 * sig2)))
    x0, y0, x1, y1 = pre["rect"][0]
    inrect = (xx // 16 >= x0) & (xx // 16 < x1) & (yy // 16 >= y0) & (yy // 16 < y1)
    a = np.where((alpha >= np.float32(1 / 255)) & inrect, alpha, 0.0)
    np.testing.assert_allclose(out["T"], 1 - a, rtol=0, atol=1e-6)
    np.testing.assert_allclose(out["rgb"][0], a * pre["rgb"][0, 0], rtol=0, atol=1e-6)


# ---- step 10b: the opacity-aware box of GS_FLAG_OBOX -------------
def test_ln_step10b_matches_the_natural_log():
    """The fixed-operation ln (atanh series) is within 2e-6 of log on [1, 255]; the box
    margin (5e-3 in ln alpha) dwarfs it."""
    ts = np.concatenate([np.linspace(1.0, 255.0, 2001), 2.0 ** np.arange(0, 8), [1.0000001, 254.9999]])
    err = max(abs(oracle.ln_step10b(float(np.float32(t))) - math.log(float(np.float32(t)))) for t in ts)
    assert err < 2e-6, err


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_obox_lists_are_an_alpha_exact_ordered_subset(name):
    """GS_FLAG_OBOX binning = the vanilla lists minus (Gaussian, tile) pairs whose alpha is
    below 1/255 on every pixel of the tile (brute force in float64 from the splats), in the
    vanilla order; Gaussians with 255*opacity < 1 are gone entirely."""
    scene, cams, bg = synth.make_config(name)
    cam = cams[0]
    pre = oracle.preprocess(scene, cam)
    pob = oracle.preprocess(scene, cam, obox=True)
    for k in ("depth", "xy", "conic", "rgb"):   # only the rect (and culling) may change
        vis = pob["touched"] > 0
        assert np.array_equal(pre[k][vis], pob[k][vis])
    assert not (pob["touched"][255.0 * pre["opacity"] < 1.0] > 0).any()
    ref = oracle.binning(pre, cam.W, cam.H)
    ob = oracle.binning(pob, cam.W, cam.H)
    assert 0 < ob["K"] < ref["K"]
    gx = (cam.W + 15) // 16
    rng = np.random.default_rng(1)
    tiles = np.nonzero(ref["ranges"][:, 1] > ref["ranges"][:, 0])[0]
    n_dropped = 0
    for t in rng.choice(tiles, min(40, len(tiles)), replace=False):
        v_all = [int(v) for v in ref["vals"][ref["ranges"][t, 0]:ref["ranges"][t, 1]]]
        v_ob = [int(v) for v in ob["vals"][ob["ranges"][t, 0]:ob["ranges"][t, 1]]]
        kept = set(v_ob)
        assert [v for v in v_all if v in kept] == v_ob
        tx, ty = t % gx, t // gx
        yy, xx = np.mgrid[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16]
        for i in v_all:
            if i in kept:
                continue
            n_dropped += 1
            dx = float(pre["xy"][i, 0]) - xx
            dy = float(pre["xy"][i, 1]) - yy
            A, B, C = (float(c) for c in pre["conic"][i])
            a = float(pre["opacity"][i]) * np.exp(-0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy)
            assert a.max() < (1.0 / 255.0) * math.exp(-0.004), (t, i, a.max())
    assert n_dropped > 0


# ---- the decision-margin mask (R-21): pins against constructed decisions -------
def _one_tile(xy, conic, opac, rgb):
    """Splats + a one-tile (16x16) binning listing every splat in order."""
    n = len(opac)
    pre = dict(xy=np.asarray(xy, np.float32).reshape(n, 2), conic=np.asarray(conic, np.float32).reshape(n, 3),
               opacity=np.asarray(opac, np.float32), rgb=np.asarray(rgb, np.float32).reshape(n, 3),
               touched=np.ones(n, np.uint32))
    b = dict(vals=np.arange(n, dtype=np.uint32), ranges=np.array([[0, n]], np.uint32), K=n)
    return pre, b


def test_margin_mask_flags_an_alpha_skip_on_the_threshold_and_bounds_its_flip():
    """A splat placed so that pixel (0,0) sits within 1e-5 of ln(1/255) in ln alpha: that
    pixel is flagged (and no decision 0.5 px away is), and the frame change caused by
    flipping the decision (opacity scaled by exp(+-3e-4), larger than the documented GPU
    error) stays within the reported flip bound."""
    s2, o = 16.0, 0.5                                   # isotropic, sigma^2 = 16
    ln_amin = math.log(float(np.float32(1.0 / 255.0)))
    d2 = 2 * s2 * (math.log(o) - ln_amin - 1e-5)        # ln alpha(0,0) = ln_amin + 1e-5
    mx = math.sqrt(d2)
    pre, b = _one_tile([[mx, 0.0]], [[1 / s2, 0.0, 1 / s2]], [o], [[1.0, 1.0, 1.0]])
    out = oracle.blend(pre, b, 16, 16)
    assert out["flag"][0, 0]
    assert out["flag"].sum() <= 2                       # only pixels on the threshold circle
    for f in (math.exp(-3e-4), math.exp(3e-4)):        # both sides of the decision
        pre2 = dict(pre, opacity=(pre["opacity"] * np.float32(f)).astype(np.float32))
        o2 = oracle.blend(pre2, b, 16, 16)
        assert abs(o2["rgb"][0, 0, 0] - out["rgb"][0, 0, 0]) <= out["bound"][0, 0] + 1e-12


def test_margin_mask_is_empty_when_no_decision_is_near_a_threshold():
    """A wide, half-transparent splat (alpha in [0.2, 0.5] on the whole tile, T far above
    1e-4): no pixel is flagged and the flip bounds are zero."""
    pre, b = _one_tile([[7.5, 7.5]], [[1e-3, 0.0, 1e-3]], [0.5], [[0.3, 0.6, 0.9]])
    out = oracle.blend(pre, b, 16, 16)
    assert not out["flag"].any() and (out["bound"] == 0).all()
    assert (out["T"] > 0.4).all()


def test_margin_mask_flags_a_termination_on_the_threshold():
    """Identical flat splats with alpha a stacked so that T after k steps is within a hair
    of 1e-4 at every pixel: the stop decision is ambiguous there, so every pixel is
    flagged; with the stack one step shorter (T far above 1e-4 at the end) nothing is."""
    k = 4
    a = 1.0 - (1e-4 * (1 + 1e-7)) ** (1.0 / k)          # T_k = 1e-4 (1 + 1e-7)
    n = k + 2
    conic = [[1e-9, 0.0, 1e-9]] * n                     # flat: alpha ~ opacity on the tile
    pre, b = _one_tile([[7.5, 7.5]] * n, conic, [a] * n, [[0.5, 0.5, 0.5]] * n)
    out = oracle.blend(pre, b, 16, 16)
    assert out["flag"].all()
    pre3, b3 = _one_tile([[7.5, 7.5]] * 2, conic[:2], [a] * 2, [[0.5, 0.5, 0.5]] * 2)
    assert not oracle.blend(pre3, b3, 16, 16)["flag"].any()


# ---- compositing readings R-2 / R-4 and the Jacobian clamp of R-14: closed forms ------
# Each of these fails under the plausible misreading it names (tests/test_oracle_mutations.py
# rebuilds the oracle with each misreading and checks that some pin fails).

def _flat(o_list, rgb_list):
    """Splats with a zero conic on one 16x16 tile: power = 0 at every pixel, so alpha = o
    exactly (Eq. 2-3 with Sigma^-1 = 0), and the list order is the given order."""
    n = len(o_list)
    return _one_tile([[7.5, 7.5]] * n, [[0.0, 0.0, 0.0]] * n, o_list, rgb_list)


def test_alpha_cap_closed_form():
    """R-4 (BASELINE.json north_star: alpha capped at 0.99; vanilla): one splat with
    o = 0.999 covering pixel (8, 8) exactly -> alpha = min(0.99, 0.999) = 0.99, so
    out = 0.99 c + 0.01 bg and T = 0.01 (PAPER.md P:169 / P:376 state no cap: without it
    T would be 1e-3). A splat with o = 0.5 is below the cap and composites at 0.5."""
    c = np.float32([0.8, 0.3, 0.1]).astype(np.float64)
    bg = np.float32([0.2, 0.4, 0.6]).astype(np.float64)
    pre, b = _one_tile([[8.0, 8.0]], [[0.05, 0.0, 0.05]], [0.999], [c])
    out = oracle.blend(pre, b, 16, 16, bg, threads=1)
    np.testing.assert_allclose(out["rgb"][:, 8, 8], 0.99 * c + 0.01 * bg, rtol=0, atol=1e-12)
    assert abs(out["T"][8, 8] - 0.01) < 1e-12
    o3, oT = oracle.blend_pixel([0], pre, 8.0, 8.0, bg)
    np.testing.assert_allclose(o3, 0.99 * c + 0.01 * bg, rtol=0, atol=1e-12)
    assert abs(oT - 0.01) < 1e-12
    pre5, b5 = _flat([0.5], [c])
    o5 = oracle.blend(pre5, b5, 16, 16, bg, threads=1)
    a = float(np.float32(0.5))
    np.testing.assert_allclose(o5["rgb"][:, 3, 11], a * c + (1 - a) * bg, rtol=0, atol=1e-12)


def test_early_termination_closed_form():
    """R-2 (BASELINE.json north_star "early termination at T < 1e-4"; vanilla): a stack of
    six flat splats with alpha = o = 0.95 gives T_j = (1 - o)^j: T_3 = 1.25e-4 >= 1e-4, and
    the 4th splat would leave T_4 = 6.25e-6 < 1e-4, so compositing stops there WITHOUT
    compositing the 4th splat: out = sum_{j<3} c_j o T_j + T_3 bg, T = T_3. Three
    misreadings give other values: compositing the stopper first (T = T_4 and its colour
    added), the paper's literal "T <= 0 -> stop" (all six composited, T = T_6), and a
    1e-6 threshold (the 4th composited, T = T_4)."""
    o = float(np.float32(0.95))
    cols = np.float32([[0.9, 0.1, 0.2], [0.1, 0.8, 0.3], [0.2, 0.2, 0.9],
                       [0.7, 0.6, 0.5], [0.3, 0.9, 0.9], [1.0, 0.0, 1.0]]).astype(np.float64)
    bg = np.float32([0.05, 0.1, 0.15]).astype(np.float64)
    pre, b = _flat([0.95] * 6, cols)
    out = oracle.blend(pre, b, 16, 16, bg, threads=1)
    T = [(1.0 - o) ** j for j in range(7)]
    assert T[3] >= 1e-4 > T[4]
    want = sum(cols[j] * o * T[j] for j in range(3)) + T[3] * bg
    for py, px in ((0, 0), (7, 9), (15, 15)):
        np.testing.assert_allclose(out["rgb"][:, py, px], want, rtol=0, atol=1e-13)
        assert abs(out["T"][py, px] - T[3]) < 1e-15
    o3, oT = oracle.blend_pixel(np.arange(6), pre, 3.0, 4.0, bg)
    np.testing.assert_allclose(o3, want, rtol=0, atol=1e-13)
    assert abs(oT - T[3]) < 1e-15
    # the same stack one splat shorter than the stop never reaches it: T = T_3 exactly too,
    # and with the stopper moved to the end of a shorter list the skip rule still holds
    pre3, b3 = _flat([0.95] * 3, cols[:3])
    o3b = oracle.blend(pre3, b3, 16, 16, bg, threads=1)
    np.testing.assert_allclose(o3b["rgb"][:, 5, 5], want, rtol=0, atol=1e-13)


def test_jacobian_clamp_closed_form():
    """R-14 (vanilla EWA): the Jacobian of the projection is evaluated at the view-space
    point with x/z and y/z clamped to +-1.3 tan(fov/2) (a clamp, not a cull). Two Gaussians
    outside that cone (x/z = 1.0 and y/z = -1.2, limit 1.3 * 0.64 = 0.832) but reaching the
    image: cov2D = J Sigma J^T + 0.3 I with the clamped J, computed here by hand in float64
    from the textbook Jacobian of (f x/z + c_x, f y/z + c_y). The unclamped Jacobian and a
    1.0 tan(fov/2) clamp both miss by > 10 %."""
    from scipy.spatial.transform import Rotation
    f, z, W = 50.0, 10.0, 64
    cam = _axis_camera(W=W, H=W, f=f, D=z)       # world z = 0 is at depth 10; R = I
    tanf = float(np.float32(W / (2 * f)))
    q = np.array([[0.9, 0.2, -0.3, 0.25], [0.8, -0.1, 0.4, 0.3]], np.float64)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scales = np.array([[2.0, 0.6, 1.2], [0.7, 1.9, 1.1]])
    means = np.array([[1.0 * z, 0.1, 0.0], [0.2, -1.2 * z, 0.0]])
    sc = _scene(means, scales, q.astype(np.float32), [0.9, 0.9], _sh_zero(2, 0), 0)
    pre = oracle.preprocess(sc, cam)
    assert (pre["touched"] > 0).all()

    def cov2d(i, lim):
        m = means[i].astype(np.float32).astype(np.float64)
        v = m + np.array([0.0, 0.0, z])                           # view space (R = I, t = (0,0,z))
        u = np.clip(v[:2] / v[2], -lim, lim)
        J = np.array([[f / v[2], 0.0, -f * u[0] / v[2]], [0.0, f / v[2], -f * u[1] / v[2]]])
        Rq = Rotation.from_quat(np.roll(q[i].astype(np.float32).astype(np.float64), -1)).as_matrix()
        s = scales[i].astype(np.float32).astype(np.float64)
        return J @ (Rq @ np.diag(s * s) @ Rq.T) @ J.T + 0.3 * np.eye(2)

    for i in range(2):
        A, B, C = pre["conic"][i].astype(np.float64)
        got = np.linalg.inv(np.array([[A, B], [B, C]]))
        want = cov2d(i, 1.3 * tanf)
        assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max(), (i, got, want)
        for wrong in (cov2d(i, np.inf), cov2d(i, 1.0 * tanf)):
            assert np.abs(wrong - want).max() > 0.1 * np.abs(want).max()


def test_single_anisotropic_gaussian_matches_scipy_density():
    """Eq. (2)-(3) with a full 2x2 conic (cross term B != 0): alpha(p) = o * N(p; mu, Sigma) /
    N(mu; mu, Sigma), the bivariate normal density of scipy.stats evaluated from the 2D
    covariance Sigma = (conic)^-1, on every pixel of a tile (alpha capped at 0.99, skipped
    below 1/255): out = alpha c + (1 - alpha) bg and T = 1 - alpha."""
    from scipy.stats import multivariate_normal
    cov = np.array([[9.0, -5.5], [-5.5, 6.0]])
    inv = np.linalg.inv(cov)
    conic = np.float32([inv[0, 0], inv[0, 1], inv[1, 1]])
    mu = np.float32([6.7, 9.2])
    o = np.float32(0.93)
    c = np.float32([0.7, 0.2, 0.5]).astype(np.float64)
    bg = np.float32([0.1, 0.1, 0.3]).astype(np.float64)
    pre, b = _one_tile([mu], [conic], [o], [c])
    out = oracle.blend(pre, b, 16, 16, bg, threads=1)
    A, B, C = conic.astype(np.float64)
    sig = np.linalg.inv(np.array([[A, B], [B, C]]))      # the covariance the fp32 conic encodes
    rv = multivariate_normal(mean=mu.astype(np.float64), cov=sig)
    yy, xx = np.mgrid[0:16, 0:16]
    dens = rv.pdf(np.stack([xx, yy], -1).astype(np.float64)) / rv.pdf(mu.astype(np.float64))
    alpha = np.minimum(0.99, float(o) * dens)
    a = np.where(alpha >= np.float32(1 / 255), alpha, 0.0)
    assert (a > 0).sum() > 50 and (a == 0).sum() > 10     # both the kept and skipped regions
    for ch in range(3):
        np.testing.assert_allclose(out["rgb"][ch], a * c[ch] + (1 - a) * bg[ch], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["T"], 1 - a, rtol=0, atol=1e-12)
    # the mirrored cross term gives a visibly different image
    pre_m, _ = _one_tile([mu], [[conic[0], -conic[1], conic[2]]], [o], [c])
    assert np.abs(oracle.blend(pre_m, b, 16, 16, bg, threads=1)["T"] - out["T"]).max() > 0.05
