"""The multi-GPU collective path on ONE GPU (needs a B200): torch.distributed.run
with one rank, NCCL process group, SS_COLLECTIVES=force (tests/nccl_selftest.py:
TrainStep through NCCL vs without collectives, equal up to float-atomic order), and bench.py's
NCCL timing path (max-over-ranks, two-bucket all-reduce) on a short run."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, timeout):
    env = dict(os.environ, SS_COLLECTIVES="force")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_train_step_through_nccl_matches_single_process():
    r = _torchrun([os.path.join(ROOT, "tests", "nccl_selftest.py")], 600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "NCCL_SELFTEST_OK" in r.stdout
