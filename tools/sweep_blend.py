"""Builds variants of libgsrender.so with different blend pipeline shapes (-D
overrides of blend.cu's constants) and, with --run, times each on C5 through
bench.py (GS_RENDER_LIB selects the variant). Build here, run on the GPU box."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2604_02120_b200", "variants")

ap = argparse.ArgumentParser()
ap.add_argument("--run", action="store_true")
ap.add_argument("--variants", default="base:;nbld3:GS_BLEND_NBLD=3;nbld4:GS_BLEND_NBLD=4;raw8:GS_BLEND_RAW=8")
ap.add_argument("--bench-args", default="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --views 32")
a = ap.parse_args()
variants = []
for v in a.variants.split(";"):
    name, defs = v.split(":")
    variants.append((name, [d for d in defs.split(",") if d]))
if not a.run:
    from paper_2604_02120_b200 import build as B
    os.makedirs(VDIR, exist_ok=True)
    for name, defs in variants:
        print(name, B.build(force=True, out=os.path.join(VDIR, f"lib_{name}.so"), defines=defs))
else:
    for name, defs in variants:
        env = dict(os.environ, GS_RENDER_LIB=os.path.join(VDIR, f"lib_{name}.so"))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *a.bench_args.split()], env=env,
                           capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            print(name, defs, round(d["value"], 1), {k: round(v, 4) for k, v in d["stage_ms_per_frame"].items()},
                  flush=True)
            ab = d.get("ab_blend") or {}
            if ab:
                print("   direct", round(ab["blend_direct_ms"], 4), "mma",
                      {b: round(v["blend_ms"], 4) for b, v in ab.get("mma_sync", {}).items()}, flush=True)
        except Exception:
            print(name, "FAILED", r.stdout[-500:], r.stderr[-2000:], flush=True)
