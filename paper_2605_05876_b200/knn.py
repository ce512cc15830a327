"""Oriented K-nearest-neighbour index (mirror of surfsplat.knn, knn.py:18-95)
on the device: csrc/knn.cu expands cube shells of a uniform grid around each
surfel."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

DEFAULT_NEIGHBORS = 8


def _grid(cloud):
    """Uniform grid over the centres: cell ~ the median surfel scale (~ the
    neighbour spacing of a surface sampling), at most 1024 cells per axis."""
    c = cloud.centers
    lo = c.min(dim=0).values
    hi = c.max(dim=0).values
    extent = float((hi - lo).max().item())
    scale = float(torch.exp(cloud.log_scales).max(dim=1).values.median().item())
    cell = max(scale, extent / 1000.0, 1e-9)
    dim = int(min(1024, max(1, int(np.ceil(extent / cell)) + 1)))
    return [float(v) for v in lo.tolist()], cell, dim


class NeighborIndex:
    """neighbors: (N, K) int64, -1 padded; mean_dist: (N,) float64 (device
    tensors).  Same construction and fallbacks as the reference."""

    def __init__(self, cloud, k: int = DEFAULT_NEIGHBORS):
        self.k = int(k)
        if not 1 <= self.k <= 16:
            raise ValueError("k must lie in [1, 16]")
        self.rebuild(cloud)

    def rebuild(self, cloud) -> None:
        n = len(cloud)
        dev = cloud.centers.device
        k = self.k
        self.size = n
        self.neighbors = torch.full((n, k), -1, device=dev, dtype=torch.int64)
        self.mean_dist = torch.zeros(n, device=dev, dtype=torch.float64)
        if n <= 1:
            self.mean_dist[:] = 1.0
            return
        lib = _lib.load()
        org, cell, dim = _grid(cloud)
        orgp, _keep = _lib.fvec(org)
        cells = torch.empty(n, device=dev, dtype=torch.int32)
        _lib.check(lib.ss_grid_cells(n, _lib.ptr(cloud.centers), orgp, cell, dim, _lib.ptr(cells), _lib.stream_ptr()),
                   "ss_grid_cells")
        sorted_cells, order = torch.sort(cells, stable=True)
        order = order.to(torch.int32).contiguous()
        sorted_cells = sorted_cells.contiguous()
        _lib.check(lib.ss_knn_oriented(n, _lib.ptr(cloud.centers), _lib.ptr(cloud.quats), _lib.ptr(order),
                                       _lib.ptr(sorted_cells), orgp, cell, dim, k, _lib.ptr(self.neighbors),
                                       _lib.ptr(self.mean_dist), _lib.stream_ptr()), "ss_knn_oriented")
