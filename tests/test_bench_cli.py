"""bench.py's command-line contract: --gpus N runs N ranks (re-launched under
torch.distributed.run when WORLD_SIZE is unset) and reports them; a WORLD_SIZE that
disagrees with --gpus fails loudly."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2"], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=3" in (r.stdout + r.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("gather", ["nccl", "fused"])
def test_bench_gpus_2_spawns_two_ranks(gather):
    """`python bench.py --gpus 2` (as the driver's BENCH command would run it, no torchrun):
    two ranks render a 16-view orbit and gather it, and rank 0's line says n_gpus 2. On this
    one-GPU box both ranks share device 0 through the test hooks (GS_BENCH_DEVICE, the gloo
    backend: NCCL refuses two ranks on one device)."""
    env = dict(os.environ, GS_BENCH_DEVICE="0", GS_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--views", "16", "--steps", "2", "--warmup", "1",
                        "--no-e2e", "--no-ab", "--no-sweep", "--no-configs", "--no-cpu-baseline", "--gather", gather,
                        "--max-keys", str(40 << 20)], env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2
    assert line["value"] > 0 and line["steps"] == 2
