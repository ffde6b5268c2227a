"""B200-native (sm_100a) forward 3DGS renderer with GEMM-compatible alpha
blending (GEMM-GS, arXiv 2604.02120).

The render path lives in hand-written CUDA kernels behind the C-ABI of
include/gs_render.h (libgsrender.so, built in-tree by build.py); this package
holds only the thin ctypes binding (_binding.py) and the seeded synthetic
input generators (synth.py).
"""
from . import synth  # noqa: F401
from ._binding import (GS_ERR_CAPACITY, GS_ERR_CUDA, GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC, GS_BLEND_TC_COLOR, GS_FLAG_STATS, GS_FLAG_SYNC, GS_FLAG_OBOX, GS_FLAG_STATIC_SCENE, GS_FLAG_TIGHT, GS_FLAG_TILE_LISTS, GS_FLAG_TIMING,  # noqa: F401
                       Context, GsError,
                       camera, load, opts, scene_to_device, scene_to_host)
