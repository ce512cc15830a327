"""Density-aware refinement scan (mirror of surfsplat.densify, densify.py:19-202).

prune (stale | isolated | floater) -> split selection (quantile of the mean
screen-space gradient over active surfels, density gate against the frozen
KNN mean distance) -> budget -> split into two children along the longer
tangent axis.  Runs on the device: the isolation test is a fixed-radius
existence query on a uniform grid (csrc/optim.cu, replacing the reference's
scipy cKDTree k=2 query), the children are written by a native kernel, and the
selection/compaction steps are device tensor ops.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .surfels import FIELDS, SurfelCloud

R_CUT = 3.0
SPLIT_QUANTILE = 0.9
SPLIT_GRAD_FLOOR = 1e-8
SPLIT_SCALE_FACTOR = 0.7


@dataclass
class DensifyStats:
    """Screen-space gradient accumulator between topology updates (densify.py:24-40)."""
    grad_sum: torch.Tensor     # (N,) float64
    view_count: torch.Tensor   # (N,) int64

    @classmethod
    def zeros(cls, n, device="cuda"):
        return cls(torch.zeros(n, device=device, dtype=torch.float64),
                   torch.zeros(n, device=device, dtype=torch.int64))

    def accumulate(self, ss_grad, touched):
        """touched: bool per surfel (BackwardResult.touched) or per-surfel
        covering-pixel counts (counted as touched when > 0)."""
        dev = self.grad_sum.device
        self.grad_sum += torch.as_tensor(ss_grad, device=dev).to(torch.float64)
        t = torch.as_tensor(touched, device=dev)
        self.view_count += (t if t.dtype == torch.bool else t > 0).to(torch.int64)

    def mean_grad(self):
        return self.grad_sum / torch.clamp(self.view_count, min=1)


def isolated_mask(cloud: SurfelCloud) -> torch.Tensor:
    """True where the nearest other centre lies beyond R_CUT * max scale
    (densify.py:118-123), via a uniform-grid fixed-radius query."""
    n = len(cloud)
    dev = cloud.centers.device
    if n <= 1:
        return torch.zeros(n, device=dev, dtype=torch.bool)
    lib = _lib.load()
    c = cloud.centers
    lo = c.min(dim=0).values
    hi = c.max(dim=0).values
    support = R_CUT * torch.exp(cloud.log_scales).max(dim=1).values
    extent = float((hi - lo).max().item())
    cell = max(float(torch.median(support).item()) * 2.0, extent / 1024.0, 1e-12)
    dim = int(min(1024, max(1, int(np.ceil(extent / cell)) + 1)))
    org, _k1 = _lib.fvec([float(v) for v in lo.tolist()])
    cells = torch.empty(n, device=dev, dtype=torch.int32)
    _lib.check(lib.ss_grid_cells(n, _lib.ptr(c), org, cell, dim, _lib.ptr(cells), _lib.stream_ptr()), "ss_grid_cells")
    sorted_cells, order = torch.sort(cells, stable=True)
    order = order.to(torch.int32).contiguous()
    sorted_cells = sorted_cells.contiguous()
    iso = torch.empty(n, device=dev, dtype=torch.uint8)
    _lib.check(lib.ss_isolation(n, _lib.ptr(c), _lib.ptr(cloud.log_scales), _lib.ptr(order), _lib.ptr(sorted_cells),
                                org, cell, dim, _lib.ptr(iso), _lib.stream_ptr()), "ss_isolation")
    return iso.bool()


def prune_keep_mask(cloud, stats, outside_mask_votes=None, front_votes=None):
    """densify.py:101-135: keep mask and removal counts by reason."""
    stale = stats.grad_sum <= 0.0
    isolated = isolated_mask(cloud)
    floater = torch.zeros_like(stale)
    if outside_mask_votes is not None and front_votes is not None:
        fv = torch.as_tensor(front_votes, device=stale.device)
        ov = torch.as_tensor(outside_mask_votes, device=stale.device)
        floater = (fv > 0) & (ov >= fv)
    remove = stale | isolated | floater
    reasons = {"stale": int(stale.sum().item()), "isolated": int((isolated & ~stale).sum().item()),
               "floater": int((floater & ~stale & ~isolated).sum().item())}
    return ~remove, reasons


def select_split(cloud, mean_grad, mean_neighbor_dist, quantile=SPLIT_QUANTILE, grad_floor=SPLIT_GRAD_FLOOR):
    """densify.py:43-57 (numpy's default linear-interpolation quantile)."""
    active = mean_grad > 0.0
    if not bool(active.any()):
        return torch.zeros(len(cloud), device=mean_grad.device, dtype=torch.bool)
    q = float(torch.quantile(mean_grad[active].to(torch.float64), quantile, interpolation="linear").item())
    thresh = max(q, grad_floor)
    max_scale = torch.exp(cloud.log_scales).max(dim=1).values.to(torch.float64)
    mnd = torch.as_tensor(mean_neighbor_dist, device=mean_grad.device, dtype=torch.float64)
    return (mean_grad >= thresh) & (max_scale > mnd)


def split_cloud(cloud: SurfelCloud, mask):
    """densify.py:60-98: layout [kept..., +children..., -children...] and the
    index map (-1 for new rows)."""
    mask = torch.as_tensor(mask, device=cloud.centers.device, dtype=torch.bool)
    keep_idx = torch.nonzero(~mask).flatten()
    split_idx = torch.nonzero(mask).flatten()
    ns, nk = int(split_idx.numel()), int(keep_idx.numel())
    parts = {k: torch.cat([getattr(cloud, k)[keep_idx], getattr(cloud, k)[split_idx], getattr(cloud, k)[split_idx]])
             for k in FIELDS}
    if ns:
        lib = _lib.load()
        parents = split_idx.to(torch.int32).contiguous()
        _lib.check(lib.ss_split_children(ns, _lib.ptr(parents), _lib.ptr(cloud.centers), _lib.ptr(cloud.quats),
                                         _lib.ptr(cloud.log_scales), _lib.ptr(parts["centers"]),
                                         _lib.ptr(parts["log_scales"]), nk, nk + ns, _lib.stream_ptr()),
                   "ss_split_children")
    out = SurfelCloud(*(parts[k].contiguous() for k in FIELDS))
    index_map = torch.cat([keep_idx, torch.full((2 * ns,), -1, device=keep_idx.device, dtype=torch.int64)])
    return out, index_map


def refine_topology(cloud, stats, mean_neighbor_dist, max_surfels, quantile=SPLIT_QUANTILE,
                    grad_floor=SPLIT_GRAD_FLOOR, outside_mask_votes=None, front_votes=None):
    """densify.py:168-202: prune then split within the surfel budget.
    Returns (cloud, index map into the input cloud with -1 for new rows, reasons)."""
    keep, reasons = prune_keep_mask(cloud, stats, outside_mask_votes, front_votes)
    kept_idx = torch.nonzero(keep).flatten()
    kept = cloud.select(kept_idx)
    mean_grad = stats.mean_grad()[kept_idx]
    mnd = torch.as_tensor(mean_neighbor_dist, device=kept_idx.device, dtype=torch.float64)[kept_idx]
    sel = select_split(kept, mean_grad, mnd, quantile, grad_floor)
    budget = int(max_surfels) - len(kept)
    n_split = int(sel.sum().item())
    if n_split > budget:
        allowed = max(budget, 0)
        if allowed == 0:
            sel = torch.zeros_like(sel)
        else:
            cand = torch.nonzero(sel).flatten()
            order = torch.sort(-mean_grad[cand], stable=True).indices
            chosen = cand[order[:allowed]]
            sel = torch.zeros_like(sel)
            sel[chosen] = True
        n_split = allowed
    new_cloud, sub_map = split_cloud(kept, sel)
    index_map = torch.where(sub_map >= 0, kept_idx[torch.clamp(sub_map, min=0)], torch.full_like(sub_map, -1))
    reasons["split"] = n_split
    return new_cloud, index_map, reasons


def mask_votes(cloud, cameras, masks):
    """densify.py:138-165: per-surfel counts of views where the centre lands
    outside the mask, and of views where it is in front of the camera."""
    dev = cloud.centers.device
    n = len(cloud)
    c = torch.cat([cloud.centers.to(torch.float64), torch.ones(n, 1, device=dev, dtype=torch.float64)], dim=1)
    outside = torch.zeros(n, device=dev, dtype=torch.int64)
    front = torch.zeros(n, device=dev, dtype=torch.int64)
    for cam, mask in zip(cameras, masks):
        m = torch.as_tensor(np.asarray(mask), device=dev)
        h, w = m.shape[:2]
        cc = c @ torch.as_tensor(cam.view, device=dev).T
        vis = -cc[:, 2] > 0.0
        front += vis.to(torch.int64)
        hom = cc @ torch.as_tensor(cam.proj, device=dev).T
        wc = hom[:, 3]
        ok = vis & (wc.abs() > 1e-12)
        safe = torch.where(ok, wc, torch.ones_like(wc))
        ndc = torch.where(ok[:, None], hom[:, :2] / safe[:, None], torch.zeros_like(hom[:, :2]))
        px = torch.round((ndc[:, 0] + 1.0) * 0.5 * cam.width - 0.5).to(torch.int64)
        py = torch.round((1.0 - ndc[:, 1]) * 0.5 * cam.height - 0.5).to(torch.int64)
        inside = ok & (px >= 0) & (px < w) & (py >= 0) & (py < h)
        hit = torch.zeros(n, device=dev, dtype=torch.bool)
        sel = torch.nonzero(inside).flatten()
        hit[sel] = m[py[sel], px[sel]] > 0
        outside += (vis & ~hit).to(torch.int64)
    return outside, front
