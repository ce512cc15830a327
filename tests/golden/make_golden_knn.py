"""Golden fixtures for the oriented-KNN / normal-consistency row (SURVEY §8f
rank 2), produced by running the REFERENCE (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_knn.py

Two seeded clouds: a noisy sphere (orientation filter mostly passes) and a
thin two-sided shell (the filter rejects the other side), plus an isolated
surfel with no compatible neighbour (fallback distance).  Stores the
reference NeighborIndex table and normal_consistency_loss outputs in
tests/golden/knn.npz; they pin oracle/oracle.py, which checks csrc/knn.cu.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from surfsplat.knn import NeighborIndex  # noqa: E402
from surfsplat.losses import normal_consistency_loss  # noqa: E402
from surfsplat.surfels import SurfelCloud, quats_from_normals  # noqa: E402


def cloud_from(centers, normals, rng):
    n = len(centers)
    q = quats_from_normals(normals)
    q = q + rng.normal(0.0, 0.05, q.shape)  # tilt the frames a little
    return SurfelCloud(centers=centers.astype(np.float32), quats=q.astype(np.float32),
                       log_scales=np.log(rng.uniform(0.01, 0.03, (n, 2))).astype(np.float32),
                       albedo_raw=np.zeros((n, 3), np.float32), metallic_raw=np.zeros(n, np.float32),
                       roughness_raw=np.zeros(n, np.float32))


def main():
    rng = np.random.default_rng(21)
    out = {}
    # noisy sphere
    d = rng.normal(size=(700, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    sphere = cloud_from(d * (1.0 + rng.normal(0, 0.01, (700, 1))), d, rng)
    # thin shell: both sides of a plate 0.02 apart, normals facing outwards, +
    # one surfel whose normal opposes everything near it
    m = 300
    xy = rng.uniform(-0.5, 0.5, (m, 2))
    top = np.c_[xy, np.full(m, 0.01)]
    bot = np.c_[xy + rng.normal(0, 0.01, (m, 2)), np.full(m, -0.01)]
    centers = np.r_[top, bot, [[2.0, 2.0, 2.0]]]
    normals = np.r_[np.tile([0, 0, 1.0], (m, 1)), np.tile([0, 0, -1.0], (m, 1)), [[0, 0, 1.0]]]
    shell = cloud_from(centers, normals, rng)
    for name, cl in (("sphere", sphere), ("shell", shell)):
        idx = NeighborIndex(cl, k=8)
        loss, g = normal_consistency_loss(cl, idx)
        for key in ("centers", "quats", "log_scales"):
            out[f"{name}_{key}"] = getattr(cl, key)
        out[f"{name}_neighbors"] = idx.neighbors
        out[f"{name}_mean_dist"] = idx.mean_dist
        out[f"{name}_nc_loss"] = np.array(loss)
        out[f"{name}_nc_grad"] = g
    np.savez_compressed(os.path.join(HERE, "knn.npz"), **out)
    print("wrote knn.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
