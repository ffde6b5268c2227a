"""Seeded parity cases shared by the GPU parity tests and the compute-sanitizer
driver (tests/sanitize_cases.py). Inputs only: no arithmetic of the method."""
import numpy as np

from paper_2604_02120_b200 import synth


def _cfg(name, n=None):
    scene, cams, bg = synth.make_config(name, n_override=n)
    return scene, cams[0], bg


def _ragged():
    """77x45 image (ragged edge tiles), object scene with SH degree 2."""
    scene = synth.object_scene(3000, 11, sh_degree=2)
    cam = synth.look_at((0.5, -0.8, -3.5), (0, 0, 0), 77, 45, 0.8)
    return scene, cam, np.array([0.2, 0.5, 0.9], np.float32)


def _adversarial():
    """Needles (anisotropy to 300), near-plane points, huge splats, border straddlers."""
    rng = np.random.default_rng(100)
    parts = []
    s1 = synth.unbounded_scene(4000, 101, sh_degree=3, aniso_cap=300.0)
    parts.append(s1)
    n = 200
    near = synth.object_scene(n, 102, sh_degree=3)
    near.means[:] = np.array([0.0, 0.0, -3.75], np.float32) + rng.normal(0, 0.05, (n, 3)).astype(np.float32)
    parts.append(near)
    huge = synth.object_scene(20, 103, sh_degree=3)
    huge.scales[:] = 0.8
    parts.append(huge)
    scene = synth.Scene(*[np.concatenate([getattr(p, f) for p in parts]) for f in
                          ("means", "scales", "rots", "opacity", "shs")], 3)
    cam = synth.look_at((0.0, 0.0, -4.0), (0, 0, 0), 160, 120, 1.0)
    return scene, cam, np.array([0.0, 0.0, 0.0], np.float32)


def _dense():
    """Tile lists longer than the shared-memory sort capacities: ~40k Gaussians in
    a few tiles (global chunked sort path) and ~8k in others (1024-thread path)."""
    rng = np.random.default_rng(104)
    a = synth.object_scene(40000, 105, sh_degree=1)
    a.means[:] = rng.normal(0.0, 0.02, (40000, 3)).astype(np.float32)
    a.scales[:] = 0.004
    b = synth.object_scene(8000, 106, sh_degree=1)
    b.means[:] = (np.array([0.9, 0.6, 0.0]) + rng.normal(0.0, 0.03, (8000, 3))).astype(np.float32)
    b.scales[:] = 0.004
    scene = synth.Scene(*[np.concatenate([getattr(p, f) for p in (a, b)]) for f in
                          ("means", "scales", "rots", "opacity", "shs")], 1)
    cam = synth.look_at((0.0, 0.0, -4.0), (0, 0, 0), 96, 96, 0.7)
    return scene, cam, np.array([0.3, 0.3, 0.3], np.float32)


def _wide(W=4200, H=40):
    """Wide / tall tile grids: 263 columns take the two-level path with 9-bit
    column digits; 525 rows (> 512) take the one-level path (all K (tile,
    index) pairs expanded, ceil(tile bits / 8) stable passes)."""
    scene = synth.object_scene(20000, 107, sh_degree=3)
    cam = synth.look_at((0.0, -0.3, -3.2), (0, 0, 0), W, H, 1.6 if W > H else 0.05)
    return scene, cam, np.array([0.1, 0.2, 0.3], np.float32)


CASES = {"C1": lambda: _cfg("C1"), "C2": lambda: _cfg("C2"), "ragged": _ragged, "adversarial": _adversarial,
         "dense": _dense, "wide": _wide, "tall": lambda: _wide(40, 8400)}
