"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no projection, no SH, no
blending). It only draws Gaussian clouds and pinhole cameras whose shapes,
sizes and value distributions follow the paper's workloads (PAPER.md Table
"3DGS Workloads Statics", lines 463-484; BASELINE.json configs) with the
recipe of SURVEY.md §8(d) / DESIGN.md "Input recipe".

Everything is numpy PCG64, float32 little-endian, activated values (scales
> 0, unit quaternions (w,x,y,z), opacity in (0,1)), exactly what the C-ABI
`gs_render` takes (include/gs_render.h).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Camera:
    """Pinhole camera, OpenCV convention (x right, y down, z forward).

    R: world->camera rotation, row-major 3x3; t: translation; a world point p
    maps to R p + t. Pixel (i, j) has its centre at integer coordinates
    (i, j) (SURVEY C-15), so the vanilla-equivalent principal point is
    ((W-1)/2, (H-1)/2). tan_fovx/tan_fovy = W/(2 fx), H/(2 fy) are given
    explicitly (they bound the Jacobian clamp, reading R-14).
    """
    R: np.ndarray
    t: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    znear: float
    tan_fovx: float
    tan_fovy: float
    campos: np.ndarray
    W: int
    H: int

    def packed(self) -> np.ndarray:
        """22 float32 in the order of `gs_camera` (include/gs_render.h)."""
        return np.concatenate([
            np.asarray(self.R, np.float32).reshape(9),
            np.asarray(self.t, np.float32).reshape(3),
            np.array([self.fx, self.fy, self.cx, self.cy, self.znear,
                      self.tan_fovx, self.tan_fovy], np.float32),
            np.asarray(self.campos, np.float32).reshape(3),
        ]).astype(np.float32)


@dataclasses.dataclass
class Scene:
    means: np.ndarray      # [N,3] f32
    scales: np.ndarray     # [N,3] f32 (activated, > 0)
    rots: np.ndarray       # [N,4] f32 unit (w,x,y,z)
    opacity: np.ndarray    # [N]   f32 in (0,1)
    shs: np.ndarray        # [N,M,3] f32, M = (deg+1)^2
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.means.shape[0])


def look_at(eye, target, W, H, fov_x, znear=0.2) -> Camera:
    """Camera at `eye` looking at `target`, world 'down' is +y (OpenCV)."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    down = np.array([0.0, 1.0, 0.0])
    r = np.cross(down, f)
    if np.linalg.norm(r) < 1e-9:
        r = np.array([1.0, 0.0, 0.0])
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f], 0)
    t = -R @ eye
    fx = W / (2.0 * math.tan(fov_x / 2.0))
    fy = fx
    return Camera(R=R.astype(np.float32), t=t.astype(np.float32), fx=float(np.float32(fx)),
                  fy=float(np.float32(fy)), cx=(W - 1) / 2.0, cy=(H - 1) / 2.0,
                  znear=znear, tan_fovx=float(np.float32(W / (2.0 * fx))),
                  tan_fovy=float(np.float32(H / (2.0 * fy))),
                  campos=eye.astype(np.float32), W=W, H=H)


def _common(rng, n, sh_degree, aniso_cap, log_scale):
    """Rotation, opacity, SH and disc-like anisotropic scales."""
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    # bimodal opacity like trained scenes: 40% near-opaque, rest diffuse
    hi = rng.random(n) < 0.4
    logit = np.where(hi, rng.normal(4.0, 1.0, n), rng.normal(-1.5, 1.5, n))
    opacity = 1.0 / (1.0 + np.exp(-logit))
    opacity = np.clip(opacity, 1e-4, 0.9999)
    ls = np.repeat(log_scale[:, None], 3, 1) + rng.normal(0.0, 0.25, (n, 3))
    ax = rng.integers(0, 3, n)
    ls[np.arange(n), ax] -= 1.5                       # one flat axis (disc-like)
    # anisotropy cap: max/min <= aniso_cap (DESIGN.md input recipe, C-11)
    lo = ls.max(1, keepdims=True) - math.log(aniso_cap)
    ls = np.maximum(ls, lo)
    scales = np.exp(ls)
    m = (sh_degree + 1) ** 2
    shs = np.empty((n, m, 3))
    shs[:, 0, :] = rng.normal(0.0, 0.6, (n, 3))
    if m > 1:
        shs[:, 1:, :] = rng.normal(0.0, 0.08, (n, m - 1, 3))
    return q, opacity, scales, shs


def object_scene(n, seed, sh_degree=3, aniso_cap=30.0) -> Scene:
    """Object-centric cloud (NeRF-synthetic shape): 64 blobs, shell points."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centres = rng.normal(0.0, 0.45, (64, 3))
    which = rng.integers(0, 64, n)
    d = rng.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rad = rng.uniform(0.15, 0.35, n)
    means = centres[which] + d * rad[:, None]
    log_scale = rng.normal(math.log(0.008), 0.5, n)
    q, op, sc, shs = _common(rng, n, sh_degree, aniso_cap, log_scale)
    return Scene(means.astype(np.float32), sc.astype(np.float32), q.astype(np.float32),
                 op.astype(np.float32), shs.astype(np.float32), sh_degree)


def unbounded_scene(n, seed, sh_degree=3, aniso_cap=30.0) -> Scene:
    """Unbounded cloud (Mip-NeRF360 / T&T / DB shape): dense centre + far shell."""
    rng = np.random.Generator(np.random.PCG64(seed))
    central = rng.random(n) < 0.65
    means = np.empty((n, 3))
    nc = int(central.sum())
    means[central] = rng.normal(0.0, 1.0, (nc, 3)) * np.array([1.5, 0.5, 1.5])
    ns = n - nc
    d = rng.standard_normal((ns, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = np.exp(rng.uniform(math.log(4.0), math.log(30.0), ns))
    means[~central] = d * r[:, None]
    dist = np.linalg.norm(means, axis=1)
    log_scale = rng.normal(math.log(0.006), 0.7, n) + np.log(np.maximum(1.0, dist / 2.0))
    q, op, sc, shs = _common(rng, n, sh_degree, aniso_cap, log_scale)
    return Scene(means.astype(np.float32), sc.astype(np.float32), q.astype(np.float32),
                 op.astype(np.float32), shs.astype(np.float32), sh_degree)


def orbit_cameras(n_views, W, H, fov_x, radius=4.0, elev_deg=20.0):
    """n_views cameras on a circle around the origin (BASELINE.json configs[4])."""
    cams = []
    el = math.radians(elev_deg)
    for k in range(n_views):
        az = 2.0 * math.pi * k / n_views
        eye = (radius * math.cos(el) * math.sin(az), -radius * math.sin(el),
               -radius * math.cos(el) * math.cos(az))
        cams.append(look_at(eye, (0.0, 0.0, 0.0), W, H, fov_x))
    return cams


# --- the BASELINE.json configurations --------------------------------------
CONFIGS = {
    # name: (builder, N, sh_degree, W, H, fov_x, eye, seed, bg)
    "C1": ("object", 1024, 0, 64, 64, 0.69, (0.0, -1.0, -4.0), 0, (0.0, 0.0, 0.0)),
    "C2": ("object", 300_000, 3, 800, 800, 0.6911, None, 1, (1.0, 1.0, 1.0)),
    "C3": ("unbounded", 5_800_000, 3, 1297, 840, 1.0, None, 2, (0.0, 0.0, 0.0)),
    "C4a": ("unbounded", 2_500_000, 3, 979, 546, 1.4, None, 3, (0.0, 0.0, 0.0)),
    "C4b": ("unbounded", 2_300_000, 3, 1264, 832, 1.2, None, 4, (0.0, 0.0, 0.0)),
    "C5": ("unbounded", 6_000_000, 3, 1920, 1080, math.radians(60.0), None, 5, (0.0, 0.0, 0.0)),
}


def make_config(name, n_override=None, views=1):
    """Returns (scene, [cameras], bg) for a BASELINE.json config."""
    kind, n, deg, W, H, fov, eye, seed, bg = CONFIGS[name]
    if n_override is not None:
        n = n_override
    scene = (object_scene if kind == "object" else unbounded_scene)(n, seed, deg)
    if eye is not None and views == 1:
        cams = [look_at(eye, (0.0, 0.0, 0.0), W, H, fov)]
    else:
        cams = orbit_cameras(views if views > 1 else (64 if name == "C5" else 1), W, H, fov)
        if views == 1:
            cams = cams[:1]
    return scene, cams, np.array(bg, np.float32)
