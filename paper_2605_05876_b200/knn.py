"""Oriented K-nearest-neighbour index (mirror of surfsplat.knn, knn.py:18-95)
on the device: a dense cell grid built on the device (csrc/grid.cu) and one
thread per surfel, in cell order, expanding cube shells of cells around it
(SURVEY §8f rank 2).  No host synchronisation."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

DEFAULT_NEIGHBORS = 8


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
        grid, dim = _lib.cell_grid(cloud.centers, n)
        # coarse grid (4x wider cells) for the queries whose k-th oriented
        # neighbour lies far away
        gridc, dimc = _lib.cell_grid(cloud.centers, n, dim=max(1, dim // 4))
        # cell-ordered normals + the deferred-query list (scratch)
        ws = torch.empty((int(lib.ss_knn_workspace_bytes(n)) + 7) // 8, device=dev, dtype=torch.float64)
        _lib.check(lib.ss_knn_dense(n, _lib.ptr(cloud.centers), _lib.ptr(cloud.quats), _lib.ptr(grid), dim,
                                    _lib.ptr(gridc), dimc, k,
                                    _lib.ptr(ws), _lib.ptr(self.neighbors), _lib.ptr(self.mean_dist),
                                    _lib.stream_ptr()),
                   "ss_knn_dense")
