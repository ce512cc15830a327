"""Data parallelism over views on CPU (gloo, world_size 2).

The multi-GPU step shards a batch of views across ranks, sums each rank's
per-view gradients locally into one packed buffer (GradPack, the same class
TrainStep uses) and all-reduces it.  Here each rank computes its views'
gradients with the CPU oracle and the all-reduced buffer must equal the
single-process sum over all views.
"""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_05876_b200.step import PARAMS, GradPack, shard_views


def _scene():
    from paper_2605_05876_b200 import scenes
    from paper_2605_05876_b200.camera import fibonacci_cameras
    gt = scenes.config0(5, 300)
    opt = scenes.perturb(gt, 6)
    cams = fibonacci_cameras(5, 3.0, 24, 24, fov_y_deg=40.0)
    return SimpleNamespace(**gt), SimpleNamespace(**opt), cams


def _view_grads(gt, opt, cam):
    from oracle import oracle as O
    target = O.render(gt, cam).rgb
    res = O.render(opt, cam)
    val, g = O.photometric_l1(res.rgb, target)
    back = O.backward_image(opt, res, g, None, 0.0)
    return val, back


def _fill(pack, gt, opt, cams, views):
    pack.zero()
    for v in views:
        val, back = _view_grads(gt, opt, cams[v])
        for k in PARAMS:
            pack.grads[k] += torch.tensor(back[k], dtype=pack.flat.dtype).reshape(pack.grads[k].shape)
        pack.grads["ss_grad"] += torch.tensor(back["ss_grad"], dtype=pack.flat.dtype)
        pack.view_count += torch.tensor(back["touched"].astype(np.float64))
        pack.loss += val


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gt, opt, cams = _scene()
    pack = GradPack(len(opt.centers), 1, "cpu", dtype=torch.float64)
    _fill(pack, gt, opt, cams, shard_views(len(cams), world, rank))
    pack.all_reduce()
    if rank == 0:
        torch.save({"flat": pack.flat.clone(), "touched": pack.view_count.clone()}, out)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_views_partition():
    for n in (1, 5, 64):
        for world in (1, 2, 3, 8):
            got = sum((shard_views(n, world, r) for r in range(world)), [])
            assert got == list(range(n))


def test_two_rank_allreduce_equals_single_process(tmp_path):
    out = str(tmp_path / "rank0.pt")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    got = torch.load(out)
    gt, opt, cams = _scene()
    ref = GradPack(len(opt.centers), 1, "cpu", dtype=torch.float64)
    _fill(ref, gt, opt, cams, range(len(cams)))
    torch.testing.assert_close(got["flat"], ref.flat, rtol=1e-12, atol=1e-15)
    assert torch.equal(got["touched"], ref.view_count) and float(ref.view_count.max()) > 1
