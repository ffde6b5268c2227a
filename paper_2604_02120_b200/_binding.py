"""Thin ctypes binding of libgsrender.so (include/gs_render.h).

Argument marshalling only: every step of the render path runs in the CUDA
kernels behind the C-ABI. Names mirror the C entry points. Device arrays are
torch CUDA tensors (PyTorch supplies device memory and streams); the host
entry point takes numpy arrays. There is no CPU fallback: if the library is
missing or the device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GS_RENDER_LIB: an alternative build of this same library (tuning sweeps, tools/sweep_blend.py)
LIB_PATH = os.environ.get("GS_RENDER_LIB") or os.path.join(_HERE, "libgsrender.so")

GS_OK = 0
GS_ERR_INVALID_ARG = -1
GS_ERR_ALIGNMENT = -2
GS_ERR_CAPACITY = -3
GS_ERR_CUDA = -4
GS_ERR_UNSUPPORTED_ARCH = -5
GS_ERR_NO_DEVICE = -6
GS_BLEND_TC = 0
GS_BLEND_DIRECT = 1
GS_BLEND_MMA = 2
GS_BLEND_TC_COLOR = 3   # N4: colour sum as a second tcgen05 product (include/gs_render.h)
GS_FLAG_SYNC = 1
GS_FLAG_TIMING = 2
GS_FLAG_STATS = 4
GS_FLAG_TIGHT = 8
GS_FLAG_OBOX = 16
GS_FLAG_STATIC_SCENE = 32
GS_FLAG_TILE_LISTS = 64

# every entry point declared in include/gs_render.h
EXPORTS = ("gs_ctx_create", "gs_ctx_destroy", "gs_render", "gs_render_views", "gs_render_views_host",
           "gs_last_stats", "gs_status_string", "gs_device_arch", "gs_debug_preprocess",
           "gs_debug_binning", "gs_debug_blend", "gs_debug_exponents", "gs_stage_times",
           "gs_debug_set_trace", "gs_set_view_group", "gs_debug_timeline", "gs_stream_wait_group",
           "gs_render_views_host_async", "gs_stream_wait_view")


class GsError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"{what}: {status_string(code)} ({code})")


class gs_camera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_float * 9), ("t", ctypes.c_float * 3), ("fx", ctypes.c_float),
                ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("znear", ctypes.c_float), ("tan_fovx", ctypes.c_float), ("tan_fovy", ctypes.c_float),
                ("campos", ctypes.c_float * 3)]


class gs_opts(ctypes.Structure):
    _fields_ = [("bg", ctypes.c_float * 3), ("sh_degree", ctypes.c_int), ("sh_stride", ctypes.c_int),
                ("scale_modifier", ctypes.c_float), ("blend", ctypes.c_int), ("flags", ctypes.c_uint),
                ("batch", ctypes.c_int), ("band", ctypes.c_int), ("n_bands", ctypes.c_int)]


class gs_stats(ctypes.Structure):
    _fields_ = [("n_points", ctypes.c_int64), ("n_visible", ctypes.c_int64), ("n_keys", ctypes.c_int64),
                ("capacity_keys", ctypes.c_int64), ("status", ctypes.c_int), ("launches", ctypes.c_int64),
                ("pairs_evaluated", ctypes.c_int64), ("pairs_kept", ctypes.c_int64)]


_lib = None


def load():
    """Loads libgsrender.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    cam_p, opt_p = ctypes.POINTER(gs_camera), ctypes.POINTER(gs_opts)
    sig = {
        "gs_ctx_create": [ctypes.POINTER(P), I, I64, I64, I, I],
        "gs_ctx_destroy": [P],
        "gs_render": [P, P, I, P, P, P, P, P, cam_p, I, I, opt_p, P, P],
        "gs_render_views": [P, P, I, P, P, P, P, P, cam_p, I, I, I, opt_p, P, P],
        "gs_render_views_host": [P, P, I, P, P, P, P, P, cam_p, I, I, I, opt_p, P, P],
        "gs_render_views_host_async": [P, P, I, P, P, P, P, P, cam_p, I, I, I, opt_p, P, P],
        "gs_last_stats": [P, ctypes.POINTER(gs_stats)],
        "gs_status_string": [I],
        "gs_device_arch": [I],
        "gs_debug_preprocess": [P, P, I, P, P, P, P, P, cam_p, I, I, opt_p, P, P, P, P, P, P, P],
        "gs_debug_binning": [P, P, I, P, P, P, P, P, cam_p, I, I, opt_p, P, P, P, I64,
                             ctypes.POINTER(I64)],
        "gs_debug_blend": [P, P, I, P, P, P, P, P, I64, P, I, I, opt_p, P, P],
        "gs_debug_exponents": [P, P, I, P, P, P, P, I64, P, I, I, P],
        "gs_stage_times": [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)],
        "gs_debug_set_trace": [P, P],
        "gs_set_view_group": [P, I, I],
        "gs_stream_wait_group": [P, P, I],
        "gs_stream_wait_view": [P, P, I],
        "gs_debug_timeline": [P, ctypes.POINTER(ctypes.c_double), I, ctypes.POINTER(I)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_char_p if name == "gs_status_string" else ctypes.c_int
    _lib = lib
    return lib


def status_string(code):
    try:
        return load().gs_status_string(int(code)).decode()
    except Exception:  # library missing: still give a readable message
        return "status"


def _check(code, what):
    if code != GS_OK:
        raise GsError(code, what)


def camera(cam) -> gs_camera:
    """synth.Camera (or any object with the same fields) -> gs_camera."""
    c = gs_camera()
    c.R[:] = [float(v) for v in np.asarray(cam.R, np.float32).reshape(9)]
    c.t[:] = [float(v) for v in np.asarray(cam.t, np.float32).reshape(3)]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.znear, c.tan_fovx, c.tan_fovy = float(cam.znear), float(cam.tan_fovx), float(cam.tan_fovy)
    c.campos[:] = [float(v) for v in np.asarray(cam.campos, np.float32).reshape(3)]
    return c


def opts(bg=(0.0, 0.0, 0.0), sh_degree=3, sh_stride=None, scale_modifier=1.0, blend=GS_BLEND_TC, flags=0,
         batch=0, band=0, n_bands=0):
    o = gs_opts()
    o.bg[:] = [float(v) for v in bg]
    o.sh_degree = int(sh_degree)
    o.sh_stride = int(sh_stride if sh_stride is not None else max(1, (sh_degree + 1) ** 2))
    o.scale_modifier = float(scale_modifier)
    o.blend = int(blend)
    o.flags = int(flags)
    o.batch = int(batch)
    o.band = int(band)
    o.n_bands = int(n_bands)
    return o


def _ptr(t):
    """Device pointer of a torch tensor (contiguous) or None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        assert t.is_contiguous(), "tensors must be contiguous"
        return ctypes.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(int(t))


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


class Context:
    """Owns a gs_ctx (device workspace) -- gs_ctx_create / gs_ctx_destroy."""

    def __init__(self, device=0, max_points=1 << 20, max_keys=1 << 24, max_w=2048, max_h=2048):
        self.lib = load()
        h = ctypes.c_void_p()
        _check(self.lib.gs_ctx_create(ctypes.byref(h), int(device), int(max_points), int(max_keys),
                                      int(max_w), int(max_h)), "gs_ctx_create")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.gs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- product entry points ----------------------------------------------
    def gs_render(self, scene_t, cam, W, H, o, out_rgb, out_T, stream=None):
        m, s, r, op, sh, n = scene_t
        _check(self.lib.gs_render(self.h, _stream(stream), n, _ptr(m), _ptr(s), _ptr(r), _ptr(op), _ptr(sh),
                                  ctypes.byref(cam), W, H, ctypes.byref(o), _ptr(out_rgb), _ptr(out_T)),
               "gs_render")

    def gs_render_views(self, scene_t, cams, W, H, o, out_rgb, out_T, stream=None):
        m, s, r, op, sh, n = scene_t
        arr = (gs_camera * len(cams))(*cams)
        _check(self.lib.gs_render_views(self.h, _stream(stream), n, _ptr(m), _ptr(s), _ptr(r), _ptr(op),
                                        _ptr(sh), arr, len(cams), W, H, ctypes.byref(o), _ptr(out_rgb),
                                        _ptr(out_T)), "gs_render_views")

    def gs_render_views_host(self, scene_np, cams, W, H, o, h_out_rgb, h_out_T, stream=None, async_=False):
        m, s, r, op, sh, n = scene_np
        arr = (gs_camera * len(cams))(*cams)
        fn = self.lib.gs_render_views_host_async if async_ else self.lib.gs_render_views_host
        _check(fn(self.h, _stream(stream), n, _ptr(m), _ptr(s), _ptr(r), _ptr(op), _ptr(sh), arr, len(cams), W, H,
                  ctypes.byref(o), _ptr(h_out_rgb), _ptr(h_out_T)), "gs_render_views_host")

    def gs_debug_timeline(self, max_spans=4096):
        """[(stage, start_ms, end_ms)] of the GS_FLAG_TIMING spans since gs_stage_times."""
        buf = (ctypes.c_double * (3 * max_spans))()
        n = ctypes.c_int(0)
        _check(self.lib.gs_debug_timeline(self.h, buf, max_spans, ctypes.byref(n)), "gs_debug_timeline")
        return [(int(buf[3 * i]), buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)]

    def gs_stream_wait_view(self, stream, v):
        """Device-side wait of `stream` (torch.cuda.Stream) until views [0, v] of the last
        gs_render_views call are complete."""
        _check(self.lib.gs_stream_wait_view(self.h, _stream(stream), int(v)), "gs_stream_wait_view")

    def gs_stream_wait_group(self, stream, g):
        """Device-side wait of `stream` (torch.cuda.Stream) for view group g of the last
        gs_render_views call."""
        _check(self.lib.gs_stream_wait_group(self.h, _stream(stream), int(g)), "gs_stream_wait_group")

    def gs_set_view_group(self, g, concurrent=True):
        _check(self.lib.gs_set_view_group(self.h, int(g), int(bool(concurrent))), "gs_set_view_group")

    def gs_last_stats(self):
        st = gs_stats()
        _check(self.lib.gs_last_stats(self.h, ctypes.byref(st)), "gs_last_stats")
        return st

    def gs_stage_times(self):
        """(preprocess_ms, binning_ms, blend_ms) summed over GS_FLAG_TIMING frames, and the frame count."""
        ms = (ctypes.c_double * 3)()
        fr = ctypes.c_int64(0)
        _check(self.lib.gs_stage_times(self.h, ms, ctypes.byref(fr)), "gs_stage_times")
        return tuple(ms), fr.value

    # --- test entry points ---------------------------------------------------
    def gs_debug_preprocess(self, scene_t, cam, W, H, o, outs, stream=None):
        m, s, r, op, sh, n = scene_t
        _check(self.lib.gs_debug_preprocess(self.h, _stream(stream), n, _ptr(m), _ptr(s), _ptr(r), _ptr(op),
                                            _ptr(sh), ctypes.byref(cam), W, H, ctypes.byref(o),
                                            *[_ptr(outs[k]) for k in ("depth", "xy", "conic", "rgb", "rect",
                                                                        "radius", "touched")]),
               "gs_debug_preprocess")

    def gs_debug_binning(self, scene_t, cam, W, H, o, keys, vals, ranges, stream=None):
        m, s, r, op, sh, n = scene_t
        nk = ctypes.c_int64(0)
        code = self.lib.gs_debug_binning(self.h, _stream(stream), n, _ptr(m), _ptr(s), _ptr(r), _ptr(op),
                                         _ptr(sh), ctypes.byref(cam), W, H, ctypes.byref(o), _ptr(keys),
                                         _ptr(vals), _ptr(ranges), int(keys.numel()), ctypes.byref(nk))
        return code, nk.value

    def gs_debug_blend(self, n, xy, conic, opacity, rgb, vals, K, ranges, W, H, o, out_rgb, out_T,
                       stream=None):
        _check(self.lib.gs_debug_blend(self.h, _stream(stream), n, _ptr(xy), _ptr(conic), _ptr(opacity),
                                       _ptr(rgb), _ptr(vals), int(K), _ptr(ranges), W, H, ctypes.byref(o),
                                       _ptr(out_rgb), _ptr(out_T)), "gs_debug_blend")

    def gs_debug_set_trace(self, trace):
        _check(self.lib.gs_debug_set_trace(self.h, _ptr(trace)), "gs_debug_set_trace")

    def gs_debug_exponents(self, n, xy, conic, opacity, vals, K, ranges, W, H, out_m, stream=None):
        _check(self.lib.gs_debug_exponents(self.h, _stream(stream), n, _ptr(xy), _ptr(conic), _ptr(opacity),
                                           _ptr(vals), int(K), _ptr(ranges), W, H, _ptr(out_m)),
               "gs_debug_exponents")


def scene_to_device(scene, device="cuda"):
    """Uploads a synth.Scene; returns the (means, scales, rots, opacity, shs, N) tuple."""
    import torch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)
    return (t(scene.means), t(scene.scales), t(scene.rots), t(scene.opacity), t(scene.shs), scene.n)


def scene_to_host(scene, pinned=True):
    """Host (optionally pinned) torch CPU tensors for gs_render_views_host, plus N."""
    import torch
    out = []
    for a in (scene.means, scene.scales, scene.rots, scene.opacity, scene.shs):
        t = torch.from_numpy(np.ascontiguousarray(a, np.float32))
        out.append(t.pin_memory() if pinned else t)
    return (*out, scene.n)
