"""Density-aware refinement scan (mirror of surfsplat.densify, densify.py:19-202).

prune (stale | isolated | floater) -> split selection (quantile of the mean
screen-space gradient over active surfels, density gate against the frozen
KNN mean distance) -> budget -> split into two children along the longer
tangent axis.  Runs on the device: the isolation test is a fixed-radius
existence query on a uniform grid (csrc/optim.cu, replacing the reference's
scipy cKDTree k=2 query), and refine_topology runs the whole pass (prune, quantile, budget,
compaction, children, optimiser-state remap) as native kernels with one host
read of the counters at the end (csrc/refine.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes

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
        """One view (densify.py:35-37): touched is BackwardResult.touched (bool
        per surfel), adding 1 to the view count of every touched surfel.

        A batched step (TrainStep) passes its summed ss_grad and its
        `view_count` -- the number of the step's views each surfel was touched
        in (a float or int count, not a bool) -- which is exactly the sum of
        the per-view accumulate() calls over those views."""
        dev = self.grad_sum.device
        self.grad_sum += torch.as_tensor(ss_grad, device=dev).to(torch.float64)
        t = torch.as_tensor(touched, device=dev)
        if t.dtype == torch.bool:
            self.view_count += t.to(torch.int64)
        else:
            self.view_count += torch.round(t.to(torch.float64)).to(torch.int64)

    def mean_grad(self):
        return self.grad_sum / torch.clamp(self.view_count, min=1)


def isolated_flags(cloud: SurfelCloud) -> torch.Tensor:
    """uint8 per surfel: 1 where the nearest other centre lies beyond
    R_CUT * max scale (densify.py:118-123).  Fixed-radius existence query on
    a dense cell grid built on the device (csrc/grid.cu): no host round trip."""
    n = len(cloud)
    dev = cloud.centers.device
    if n <= 1:
        return torch.zeros(n, device=dev, dtype=torch.uint8)
    lib = _lib.load()
    grid, dim = _lib.cell_grid(cloud.centers, n)
    iso = torch.empty(n, device=dev, dtype=torch.uint8)
    _lib.check(lib.ss_isolation_dense(n, _lib.ptr(cloud.centers), _lib.ptr(cloud.log_scales), _lib.ptr(grid), dim,
                                      _lib.ptr(iso), _lib.stream_ptr()), "ss_isolation_dense")
    return iso


def isolated_mask(cloud: SurfelCloud) -> torch.Tensor:
    """True where the nearest other centre lies beyond R_CUT * max scale
    (densify.py:118-123)."""
    return isolated_flags(cloud).bool()


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


_ROLES = {"centers": 2, "log_scales": 3}
LAST_REFINE = {}  # diagnostics of the last refine_topology call (kept, active, candidates, threshold)


def refine_topology(cloud, stats, mean_neighbor_dist, max_surfels, quantile=SPLIT_QUANTILE,
                    grad_floor=SPLIT_GRAD_FLOOR, outside_mask_votes=None, front_votes=None, optimizer=None):
    """densify.py:168-202: prune then split within the surfel budget.
    Returns (cloud, index map into the input cloud with -1 for new rows,
    reasons).

    Runs as device kernels (csrc/refine.cu): isolation query, prune flags,
    numpy-'linear' quantile by radix select, candidate and budget selection,
    compaction and the new rows -- one host read of the counters at the end.
    With `optimizer` (an Adam), its state rows are remapped in the same pass
    (Adam.remap of every parameter, adam.py:43-58)."""
    lib = _lib.load()
    n = len(cloud)
    dev = cloud.centers.device
    s = _lib.stream_ptr()
    gs = torch.as_tensor(stats.grad_sum, device=dev).to(torch.float64).contiguous()
    vc = torch.as_tensor(stats.view_count, device=dev).to(torch.int64).contiguous()
    mnd = torch.as_tensor(mean_neighbor_dist, device=dev).to(torch.float64).contiguous()
    if outside_mask_votes is not None and front_votes is not None:
        ov = torch.as_tensor(outside_mask_votes, device=dev).to(torch.int64).contiguous()
        fv = torch.as_tensor(front_votes, device=dev).to(torch.int64).contiguous()
    else:
        ov = fv = None
    iso = isolated_flags(cloud)
    ws = torch.empty(int(lib.ss_refine_workspace_bytes(n)), device=dev, dtype=torch.uint8)
    dst = torch.empty(n, device=dev, dtype=torch.int32)
    kind = torch.empty(n, device=dev, dtype=torch.uint8)
    counts = torch.zeros(9, device=dev, dtype=torch.int64)
    _lib.check(lib.ss_refine_plan(n, _lib.ptr(gs), _lib.ptr(vc), _lib.ptr(iso), _lib.ptr(ov), _lib.ptr(fv),
                                  _lib.ptr(cloud.log_scales), _lib.ptr(mnd), int(max_surfels), float(quantile),
                                  float(grad_floor), _lib.ptr(dst), _lib.ptr(kind), _lib.ptr(counts), _lib.ptr(ws), s),
               "ss_refine_plan")
    # outputs sized for the largest possible result (kept + splits <= max(n, max_surfels)),
    # so the new rows are written before the counts are read back
    cap = max(n, int(max_surfels), 1)
    tensors = []
    for k in FIELDS:
        t = getattr(cloud, k)
        tensors.append((t, torch.empty((cap,) + tuple(t.shape[1:]), device=dev, dtype=t.dtype), _ROLES.get(k, 0)))
    opt_new = {}
    if optimizer is not None:
        for name in list(optimizer.m):
            if name not in FIELDS:  # per-surfel state only (not the env)
                continue
            for store in (optimizer.m, optimizer.v, getattr(optimizer, "p64", {})):
                if name not in store:
                    continue
                t = store[name]
                if t.shape[0] != n:
                    raise ValueError(f"optimizer state {name!r} has {t.shape[0]} rows, the cloud {n}")
                out = torch.empty((cap,) + tuple(t.shape[1:]), device=dev, dtype=t.dtype)
                tensors.append((t, out, 1))
                opt_new[(id(store), name)] = out
    if len(tensors) > 32:
        raise ValueError("too many tensors to remap in one pass")
    index_map = torch.empty(cap, device=dev, dtype=torch.int64)
    m = len(tensors)
    src = (ctypes.c_void_p * m)(*[t[0].data_ptr() for t in tensors])
    out = (ctypes.c_void_p * m)(*[t[1].data_ptr() for t in tensors])
    rb = (ctypes.c_int * m)(*[t[0].element_size() * (t[0].numel() // max(t[0].shape[0], 1)) for t in tensors])
    roles = (ctypes.c_int * m)(*[t[2] for t in tensors])
    _lib.check(lib.ss_refine_apply(n, _lib.ptr(kind), _lib.ptr(dst), _lib.ptr(cloud.centers), _lib.ptr(cloud.quats),
                                   _lib.ptr(cloud.log_scales), m, src, out, rb, roles, _lib.ptr(index_map),
                                   _lib.ptr(ws), s), "ss_refine_apply")
    c = counts.cpu().numpy()  # the one host synchronisation
    n_out = int(c[0])
    new = SurfelCloud(*(tensors[i][1][:n_out] for i in range(len(FIELDS))))
    if optimizer is not None:
        p64 = getattr(optimizer, "p64", {})
        for name in list(optimizer.m):
            for store in (optimizer.m, optimizer.v, p64):
                key = (id(store), name)
                if key in opt_new:
                    store[name] = opt_new[key][:n_out]
            if name in p64 and (id(p64), name) in opt_new:
                # float64 masters: survivors keep theirs, new rows (zeroed
                # like the moments) take the new float32 parameters
                fresh = index_map[:n_out] < 0
                p64[name][fresh] = getattr(new, name)[fresh].to(torch.float64)
    reasons = {"stale": int(c[3]), "isolated": int(c[4]), "floater": int(c[5]), "split": int(c[2])}
    LAST_REFINE.update(kept=int(c[1]), active=int(c[6]), candidates=int(c[7]),
                       threshold=float(np.array([c[8]], dtype=np.int64).view(np.float64)[0]))
    return new, index_map[:n_out], reasons


def refine_topology_reference_order(cloud, stats, mean_neighbor_dist, max_surfels, quantile=SPLIT_QUANTILE,
                                    grad_floor=SPLIT_GRAD_FLOOR, outside_mask_votes=None, front_votes=None):
    """The same pass composed from the API-level helpers below (prune_keep_mask,
    select_split, split_cloud: device tensor ops with host reads), kept as a
    cross-check of the fused kernels."""
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
