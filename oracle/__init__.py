"""CPU oracle for the GEMM-GS forward render path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package. The product package
(paper_2604_02120_b200) never imports it and shares no code with it.

The arithmetic lives in oracle.c (fp32 preprocess in the order of
docs/preprocess_order.md, plain-definition binning, float64 blending); this
module only builds/loads the shared library and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-pthread"]


def build(force=False):
    """Compile oracle.c -> liboracle.so (gcc, no FMA contraction, no fast math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cam(ctypes.Structure):
    _fields_ = [("R", ctypes.c_float * 9), ("t", ctypes.c_float * 3),
                ("fx", ctypes.c_float), ("fy", ctypes.c_float),
                ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("znear", ctypes.c_float), ("tan_fovx", ctypes.c_float),
                ("tan_fovy", ctypes.c_float), ("campos", ctypes.c_float * 3)]


def _load():
    global _lib
    if _lib is None:
        # ORACLE_LIB: a deliberately mis-built oracle (tests/test_oracle_mutations.py only)
        path = os.environ.get("ORACLE_LIB") or build()
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        lib.orc_preprocess.restype = ctypes.c_int
        lib.orc_preprocess.argtypes = [ctypes.c_int, P, P, P, P, P, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_float, ctypes.POINTER(_Cam), ctypes.c_int,
                                       ctypes.c_int, P, P, P, P, P, P, P]
        lib.orc_preprocess_mode.restype = ctypes.c_int
        lib.orc_preprocess_mode.argtypes = lib.orc_preprocess.argtypes + [ctypes.c_int]
        lib.orc_ln_step10b.restype = ctypes.c_float
        lib.orc_ln_step10b.argtypes = [ctypes.c_float]
        lib.orc_binning.restype = ctypes.c_int64
        lib.orc_binning.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, ctypes.c_int, P, P, P,
                                    ctypes.c_int64]
        lib.orc_blend.restype = None
        lib.orc_blend.argtypes = [P, P, P, P, P, P, ctypes.c_int, ctypes.c_int, P,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_int, P, P, P, P, P]
        lib.orc_blend_pixel.restype = None
        lib.orc_blend_pixel.argtypes = [ctypes.c_int, P, P, P, P, P, ctypes.c_double,
                                        ctypes.c_double, P, P, P]
        lib.orc_vg.restype = None
        lib.orc_vg.argtypes = [ctypes.c_double] * 5 + [P]
        lib.orc_vp.restype = None
        lib.orc_vp.argtypes = [ctypes.c_double] * 2 + [P]
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def camera_struct(cam):
    c = _Cam()
    c.R[:] = [float(v) for v in np.asarray(cam.R, np.float32).reshape(9)]
    c.t[:] = [float(v) for v in np.asarray(cam.t, np.float32).reshape(3)]
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.znear, c.tan_fovx, c.tan_fovy = cam.znear, cam.tan_fovx, cam.tan_fovy
    c.campos[:] = [float(v) for v in np.asarray(cam.campos, np.float32).reshape(3)]
    return c


def preprocess(scene, cam, W=None, H=None, scale_modifier=1.0, obox=False):
    """Stage (a) per docs/preprocess_order.md (obox: with step 10b, the opacity-aware box
    of GS_FLAG_OBOX). Returns a dict of numpy arrays."""
    lib = _load()
    W = cam.W if W is None else W
    H = cam.H if H is None else H
    n = scene.n
    means, scales, rots, op = map(_c32, (scene.means, scene.scales, scene.rots, scene.opacity))
    shs = _c32(scene.shs)
    deg = scene.sh_degree
    stride = shs.shape[1] if shs.ndim == 3 else 1
    out = dict(depth=np.zeros(n, np.float32), xy=np.zeros((n, 2), np.float32),
               conic=np.zeros((n, 3), np.float32), rgb=np.zeros((n, 3), np.float32),
               rect=np.zeros((n, 4), np.int32), radius=np.zeros(n, np.int32),
               touched=np.zeros(n, np.uint32))
    c = camera_struct(cam)
    nv = lib.orc_preprocess_mode(n, _p(means), _p(scales), _p(rots), _p(op), _p(shs), deg, stride,
                                 scale_modifier, ctypes.byref(c), W, H, _p(out["depth"]), _p(out["xy"]),
                                 _p(out["conic"]), _p(out["rgb"]), _p(out["rect"]), _p(out["radius"]),
                                 _p(out["touched"]), int(bool(obox)))
    out["n_visible"] = nv
    out["opacity"] = op
    return out


def ln_step10b(t):
    """docs/preprocess_order.md step 10b: the fixed-operation ln used by GS_FLAG_OBOX."""
    return float(_load().orc_ln_step10b(float(t)))


def binning(pre, W, H):
    """Stages (b)+(c): sorted keys (tile<<32 | depth bits), vals, ranges [tiles,2]."""
    lib = _load()
    n = pre["depth"].shape[0]
    gx, gy = (W + 15) // 16, (H + 15) // 16
    K = int(pre["touched"].astype(np.int64).sum())
    keys = np.zeros(max(K, 1), np.uint64)
    vals = np.zeros(max(K, 1), np.uint32)
    ranges = np.zeros((gx * gy, 2), np.uint32)
    k2 = lib.orc_binning(n, _p(pre["depth"]), _p(pre["rect"]), _p(pre["touched"]), W, H,
                         _p(keys), _p(vals), _p(ranges), K)
    assert k2 == K
    return dict(keys=keys[:K], vals=vals[:K], ranges=ranges, K=K)


# Documented bound on the GPU's |d ln alpha| per (Gaussian, pixel) pair (R-21):
# delta = DELTA_0 + EPS_REL * S, S = the magnitude of the Eq. (6) terms summed about the
# tile centre. Measured on the B200 over every parity case (profiles/r2_precision.json):
# max |d ln alpha| <= 2.3e-6 + 1.44e-7 S; the constants carry a 1.7x / 3.3x margin.
DELTA_0 = 4e-6
EPS_REL = 2.0 ** -21
# A pixel is flagged when the summed first-order impacts of its ambiguous decisions exceed
# this (half the 2e-3 pixel gate), so an unflagged pixel's flips move it by at most 1e-3.
IMPACT_BUDGET = 1e-3


def blend(pre, binned, W, H, bg=(0.0, 0.0, 0.0), threads=None, delta0=DELTA_0, eps_rel=EPS_REL,
          budget=IMPACT_BUDGET, mask=True):
    """Stage (d) in float64. Returns rgb [3,H,W], T [H,W], flag [H,W], bound [H,W], stats."""
    lib = _load()
    threads = threads or os.cpu_count() or 1
    bg = np.asarray(bg, np.float32)
    out_rgb = np.zeros((3, H, W), np.float64)
    out_T = np.zeros((H, W), np.float64)
    flag = np.zeros((H, W), np.uint8)
    bound = np.zeros((H, W), np.float64)
    stats = np.zeros(2, np.int64)
    vis = pre["touched"] > 0
    cmax = float(max(np.abs(pre["rgb"][vis]).max(initial=0.0), np.abs(bg).max()))
    vals = binned["vals"] if binned["K"] > 0 else np.zeros(1, np.uint32)
    lib.orc_blend(_p(pre["xy"]), _p(pre["conic"]), _p(_c32(pre["opacity"])), _p(pre["rgb"]),
                  _p(vals), _p(np.ascontiguousarray(binned["ranges"])), W, H, _p(bg),
                  delta0, eps_rel, budget, cmax, int(threads), _p(out_rgb), _p(out_T),
                  _p(flag) if mask else None, _p(bound) if mask else None, _p(stats))
    return dict(rgb=out_rgb, T=out_T, flag=flag.astype(bool), bound=bound,
                evaluated=int(stats[0]), live=int(stats[1]))


def blend_pixel(order, pre, px, py, bg=(0.0, 0.0, 0.0)):
    lib = _load()
    order = np.ascontiguousarray(order, np.uint32)
    bg = np.asarray(bg, np.float32)
    o3 = np.zeros(3, np.float64)
    oT = np.zeros(1, np.float64)
    lib.orc_blend_pixel(len(order), _p(order) if len(order) else None, _p(pre["xy"]),
                        _p(pre["conic"]), _p(_c32(pre["opacity"])), _p(pre["rgb"]), float(px),
                        float(py), _p(bg), _p(o3), _p(oT))
    return o3, float(oT[0])


def vg(A, B, C, xh, yh):
    v = np.zeros(6, np.float64)
    _load().orc_vg(A, B, C, xh, yh, _p(v))
    return v


def vp(xb, yb):
    v = np.zeros(6, np.float64)
    _load().orc_vp(xb, yb, _p(v))
    return v


def render(scene, cam, bg=(0.0, 0.0, 0.0), threads=None, mask=True, obox=False, scale_modifier=1.0):
    """Whole path: preprocess -> binning -> blend."""
    pre = preprocess(scene, cam, scale_modifier=scale_modifier, obox=obox)
    b = binning(pre, cam.W, cam.H)
    out = blend(pre, b, cam.W, cam.H, bg, threads=threads, mask=mask)
    return pre, b, out
