"""Precision of the tensor-core exponent (TF32 hi/lo, K = 16, reading R-11) on the
parity cases: |d ln alpha| over the oracle's kept pairs against the magnitude S of the
Eq. (6) terms the GEMM sums (tests/gpu_util.exponent_errors). Writes a JSON summary
(max error, max error / S, percentiles, the error split by S) to argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from gpu_util import exponent_errors, make_ctx  # noqa: E402
from paper_2604_02120_b200 import synth  # noqa: E402
from test_gpu_parity import CASES  # noqa: E402

out = {}
for name in ("C1", "C2", "ragged", "adversarial", "dense", "C5"):
    if name == "C5":
        scene, cams, bg = synth.make_config("C5")
        cam = cams[0]
    else:
        scene, cam, bg = CASES[name]()
    ctx = make_ctx(scene, cam, max_keys=64 << 20)
    pre = oracle.preprocess(scene, cam)
    b = oracle.binning(pre, cam.W, cam.H)
    nt = len(b["ranges"])
    rng = np.random.default_rng(0)
    tiles = np.arange(nt) if nt <= 200 else rng.choice(nt, 96, replace=False)
    err, S = exponent_errors(ctx, scene.n, pre, b, cam.W, cam.H, tiles)
    ratio = err / np.maximum(S, 1e-30)
    bins = {}
    for lo, hi in ((0, 10), (10, 100), (100, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e9)):
        sel = (S >= lo) & (S < hi)
        if sel.any():
            bins[f"S_{lo:g}_{hi:g}"] = {"pairs": int(sel.sum()), "max_err": float(err[sel].max()),
                                        "p99_err": float(np.quantile(err[sel], 0.99))}
    out[name] = {"pairs": int(err.size), "max_err": float(err.max()), "p99_err": float(np.quantile(err, 0.99)),
                 "p999_err": float(np.quantile(err, 0.999)), "max_S": float(S.max()),
                 "max_err_over_S": float(ratio.max()), "max_err_minus_2e-22S": float((err - 2.0 ** -22 * S).max()),
                 "by_S": bins}
    print(name, json.dumps(out[name]), flush=True)
    ctx.close()
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "precision.json", "w"), indent=1)
