"""bench.py's multi-rank path on one GPU: `--gpus 2` relaunches itself under
torch.distributed.run (two ranks, gloo so both can share cuda:0), splits the
global batch (strong scaling), all-reduces the gradient bucket every step and
prints one JSON line with the weak-scaling figure next to it."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_strong_scaling_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", "--steps", "3",
           "--warmup", "3", "--T", "256", "--B", "16", "--C", "128", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 16 and d["config"]["B_per_gpu"] == 8
    assert d["weak"]["scaling"] == "weak" and d["weak"]["B_per_gpu"] == 16
    assert d["value"] > 0 and d["gpu_launches"] > 0


def test_bench_rejects_mismatched_world_size():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 2
