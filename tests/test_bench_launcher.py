"""bench.py's multi-rank launch on CPU: `bench.py --gpus N` without torchrun
re-executes itself under torch.distributed.run with N ranks; --dry-run runs
the same view sharding and two-bucket all-reduce as the GPU step over gloo."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 3])
def test_self_launch_spawns_n_ranks(n):
    d = _run("--gpus", str(n), "--dry-run")
    assert d["n_gpus"] == n and d["backend"] == "gloo"
    assert sum(d["views_per_rank"]) == 64 and max(d["views_per_rank"]) - min(d["views_per_rank"]) <= 1
    assert d["allreduce_ok"]


def test_single_rank_dry_run():
    d = _run("--dry-run")
    assert d["n_gpus"] == 1 and d["views_per_rank"] == [64] and d["allreduce_ok"]
