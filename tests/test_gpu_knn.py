"""Oriented KNN index and normal-consistency loss on the device (csrc/knn.cu)
against the reference goldens, the brute-force oracle and, at 1M surfels,
brute-force rows computed on the GPU (needs a B200)."""

import os

import numpy as np
import pytest
import torch

from parity import grad_close, host
from oracle import oracle as O

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "knn.npz")


def _cloud(centers, quats, log_scales):
    n = len(centers)
    z = np.zeros(n, np.float32)
    return ss.SurfelCloud(centers=np.asarray(centers, np.float32), quats=np.asarray(quats, np.float32),
                          log_scales=np.asarray(log_scales, np.float32), albedo_raw=np.zeros((n, 3), np.float32),
                          metallic_raw=z, roughness_raw=z)


@pytest.mark.parametrize("name", ["sphere", "shell"])
def test_knn_matches_reference_goldens(name):
    d = np.load(GOLD)
    cl = _cloud(d[f"{name}_centers"], d[f"{name}_quats"], d[f"{name}_log_scales"])
    idx = ss.NeighborIndex(cl, k=8)
    np.testing.assert_array_equal(host(idx.neighbors), d[f"{name}_neighbors"])
    np.testing.assert_allclose(host(idx.mean_dist), d[f"{name}_mean_dist"], rtol=1e-14, atol=0)
    loss, g = ss.normal_consistency_loss(cl, idx)
    assert loss == pytest.approx(float(d[f"{name}_nc_loss"]), rel=1e-12)
    assert grad_close(g, d[f"{name}_nc_grad"], rel=1e-6, floor=1e-7)[0] == 0


@pytest.mark.parametrize("k", [1, 8, 16])
def test_knn_matches_oracle(k):
    g = scenes.config2(4, 4000)
    cl = ss.SurfelCloud(**g)
    idx = ss.NeighborIndex(cl, k=k)
    nb, md = O.knn_oriented(g["centers"], g["quats"], k=k)
    np.testing.assert_array_equal(host(idx.neighbors), nb)
    np.testing.assert_allclose(host(idx.mean_dist), md, rtol=1e-14, atol=0)
    loss, gq = ss.normal_consistency_loss(cl, idx)
    rl, rg = O.normal_consistency(g["centers"], g["quats"], nb, md)
    assert loss == pytest.approx(rl, rel=1e-12)
    assert grad_close(gq, rg, rel=1e-6, floor=1e-7)[0] == 0


@pytest.mark.parametrize("k", [8, 16])
def test_knn_deferred_queries_match_oracle(k):
    """Surfels facing against their surroundings have their oriented
    neighbours far away: those queries leave the shell search for the
    whole-cloud pass (knn_brute_kernel); rows still equal the oracle's."""
    g = scenes.config2(4, 4000)
    q = g["quats"].copy()
    flip = np.random.default_rng(3).choice(len(q), 25, replace=False)
    w, x, y, z = q[flip].T
    q[flip] = np.stack([-x, w, z, -y], 1)  # q * (0, 1, 0, 0): the normal reversed
    g["quats"] = q.astype(np.float32)
    idx = ss.NeighborIndex(ss.SurfelCloud(**g), k=k)
    nb, md = O.knn_oriented(g["centers"], g["quats"], k=k)
    np.testing.assert_array_equal(host(idx.neighbors), nb)
    np.testing.assert_allclose(host(idx.mean_dist), md, rtol=1e-14, atol=0)


@pytest.mark.parametrize("n,amp,octaves", [(1_000_000, 0.08, 3), (4_000_000, 0.12, 5)])
def test_knn_full_size_rows(n, amp, octaves):
    """1M surfels (BASELINE config 2 geometry) and 4M (config 4: the grid's
    dim cap, 408 cells per axis): sampled rows equal a GPU brute force over
    all surfels."""
    g = scenes.config2(0, n, amp=amp, octaves=octaves)
    cl = ss.SurfelCloud(**g)
    idx = ss.NeighborIndex(cl, k=8)
    c = cl.centers.double()
    q = cl.quats.double()
    q = q / q.norm(dim=1, keepdim=True)
    w, x, y, z = q.unbind(1)
    nrm = torch.stack([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)], 1)
    rows = torch.from_numpy(np.random.default_rng(0).choice(len(cl), 300, replace=False)).cuda()
    nb = idx.neighbors[rows]
    for t, i in enumerate(rows.tolist()):
        d = torch.sqrt(((c - c[i]) ** 2).sum(1))
        d[i] = float("inf")
        ok = (nrm @ nrm[i]) > 0
        d = torch.where(ok, d, torch.full_like(d, float("inf")))
        top = torch.topk(d, 8, largest=False)
        assert torch.equal(nb[t].sort().values, top.indices.sort().values), i
        assert float(idx.mean_dist[i]) == pytest.approx(float(top.values.mean()), rel=1e-12)


def test_knn_degenerate_sizes():
    one = _cloud(np.zeros((1, 3)), [[1, 0, 0, 0]], np.zeros((1, 2)))
    idx = ss.NeighborIndex(one, k=4)
    assert int(idx.neighbors.max()) == -1 and float(idx.mean_dist[0]) == 1.0
    # two surfels facing away: no compatible neighbour -> nearest-point distance
    two = _cloud([[0, 0, 0], [0.3, 0, 0]], [[1, 0, 0, 0], [0, 1, 0, 0]], np.zeros((2, 2)))
    idx = ss.NeighborIndex(two, k=4)
    assert int(idx.neighbors.max()) == -1
    assert host(idx.mean_dist) == pytest.approx([0.3, 0.3], rel=1e-7)
