"""The refinement scan as device kernels (csrc/refine.cu) vs the oracle's
restatement of refine_topology (densify.py:168-202) at 120k surfels: prune
reasons, the numpy-'linear' quantile threshold (bit-exact), the budget cut
with ties, the index map, the children and the remapped Adam state."""

import numpy as np
import pytest
import torch

from parity import host

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_05876_b200 import densify, scenes  # noqa: E402
from paper_2605_05876_b200.surfels import FIELDS  # noqa: E402


def _case(n, seed, ties=False):
    rng = np.random.default_rng(seed)
    cl = scenes.config2(seed, n)
    # a few surfels far from the surface: isolated
    cl["centers"][:50] += rng.normal(0, 3.0, (50, 3)).astype(np.float32)
    grad_sum = rng.exponential(1e-4, n)
    grad_sum[rng.uniform(size=n) < 0.1] = 0.0                       # stale
    view_count = rng.integers(0, 9, n).astype(np.int64)
    if ties:  # many equal mean gradients around the cut
        grad_sum[: n // 4] = 3e-4
        view_count[: n // 4] = 1
    mnd = np.exp(rng.normal(np.log(0.004), 0.5, n))
    front = rng.integers(0, 5, n).astype(np.int64)
    outside = np.minimum(front, rng.integers(0, 7, n)).astype(np.int64)
    return cl, grad_sum, view_count, mnd, outside, front


def _expected(cl, grad_sum, view_count, mnd, max_surfels, q, outside=None, front=None):
    keep, split_rows, index_map, reasons = O.refine_topology(
        cl["centers"], cl["quats"], cl["log_scales"], grad_sum, view_count, mnd, max_surfels, quantile=q,
        outside_votes=outside, front_votes=front)
    kept_idx = np.flatnonzero(keep)
    parents = kept_idx[split_rows]
    cp, cm, cls = O.split_children(cl["centers"], cl["quats"], cl["log_scales"], parents)
    stay = index_map[index_map >= 0]
    out = {k: np.concatenate([cl[k][stay], cl[k][parents], cl[k][parents]]) for k in FIELDS}
    ns = len(parents)
    out["centers"][len(stay):len(stay) + ns] = cp
    out["centers"][len(stay) + ns:] = cm
    out["log_scales"][len(stay):] = np.concatenate([cls, cls])
    return out, index_map, reasons


@pytest.mark.parametrize("budget,ties,votes", [(1.10, False, False), (1.001, False, True), (0.95, True, False),
                                               (1.02, True, True)])
def test_refine_matches_oracle(budget, ties, votes):
    n = 120_000
    cl, grad_sum, view_count, mnd, outside, front = _case(n, 3, ties)
    max_surfels = int(budget * n)
    q = 0.95
    ov, fv = (outside, front) if votes else (None, None)
    want, want_map, want_reasons = _expected(cl, grad_sum, view_count, mnd, max_surfels, q, ov, fv)
    cloud = ss.SurfelCloud(**cl)
    stats = ss.DensifyStats(torch.tensor(grad_sum, device="cuda"), torch.tensor(view_count, device="cuda"))
    new, index_map, reasons = ss.refine_topology(cloud, stats, torch.tensor(mnd, device="cuda"), max_surfels,
                                                 quantile=q, outside_mask_votes=ov, front_votes=fv)
    for k in ("stale", "isolated", "floater", "split"):
        assert reasons[k] == want_reasons[k], (k, reasons, want_reasons)
    assert densify.LAST_REFINE["threshold"] == want_reasons["threshold"]  # bit-exact numpy quantile
    np.testing.assert_array_equal(host(index_map), want_map)
    for k in FIELDS:
        if k in ("centers", "log_scales"):
            np.testing.assert_allclose(host(getattr(new, k)), want[k], rtol=1e-6, atol=1e-7, err_msg=k)
        else:
            np.testing.assert_array_equal(host(getattr(new, k)), want[k], err_msg=k)


def test_refine_remaps_adam_state():
    """refine_topology(optimizer=...) remaps the moments like Adam.remap
    (adam.py:43-58): surviving rows follow their source, children start at 0."""
    n = 20_000
    cl, grad_sum, view_count, mnd, _, _ = _case(n, 5)
    cloud = ss.SurfelCloud(**cl)
    opt = ss.Adam()
    rng = np.random.default_rng(1)
    for k in FIELDS:
        g = torch.tensor(rng.normal(size=getattr(cloud, k).shape), device="cuda", dtype=torch.float32)
        opt.step(k, getattr(cloud, k), g, 1e-6)
    before = {k: (opt.m[k].clone(), opt.v[k].clone()) for k in FIELDS}
    stats = ss.DensifyStats(torch.tensor(grad_sum, device="cuda"), torch.tensor(view_count, device="cuda"))
    new, imap, reasons = ss.refine_topology(cloud, stats, torch.tensor(mnd, device="cuda"), int(1.05 * n),
                                            quantile=0.9, optimizer=opt)
    assert reasons["split"] > 0
    ref = ss.Adam()
    for k in FIELDS:
        ref.m[k], ref.v[k] = before[k][0].clone(), before[k][1].clone()
        ref.t[k] = 1
        ref.remap(k, imap)
        assert torch.equal(opt.m[k], ref.m[k]) and torch.equal(opt.v[k], ref.v[k]), k
        assert opt.m[k].shape[0] == len(new)


def test_refine_with_nothing_active_or_no_budget():
    n = 5000
    cl, grad_sum, view_count, mnd, _, _ = _case(n, 7)
    cloud = ss.SurfelCloud(**cl)
    zero = ss.DensifyStats(torch.zeros(n, device="cuda", dtype=torch.float64),
                           torch.zeros(n, device="cuda", dtype=torch.int64))
    new, imap, reasons = ss.refine_topology(cloud, zero, torch.tensor(mnd, device="cuda"), 2 * n)
    assert len(new) == 0 and reasons["stale"] == n and reasons["split"] == 0
    stats = ss.DensifyStats(torch.tensor(grad_sum, device="cuda"), torch.tensor(view_count, device="cuda"))
    new, imap, reasons = ss.refine_topology(cloud, stats, torch.tensor(mnd, device="cuda"), 10)
    assert reasons["split"] == 0 and len(new) == n - reasons["stale"] - reasons["isolated"]


def test_train_step_refines_every_step():
    """Config-4 style loop at small size: step -> refine (q = 0.95) ->
    rebuild the neighbour index -> next step on the new cloud; the step's
    refinement equals refine_topology on the same state."""
    gt = scenes.config2(0, 6000, amp=0.12, octaves=5)
    init = scenes.perturb(gt, 1)
    env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 2))
    cams = ss.fibonacci_cameras(4, 3.5, 96, 64)
    targets = [ss.render(ss.SurfelCloud(**gt), c, ss.RenderOptions(), env=env).rgb.contiguous() for c in cams]
    cloud = ss.SurfelCloud(**init)
    ts = ss.TrainStep(cloud, env, 96, 64, surfel_capacity=7000)
    index = ss.NeighborIndex(ts.cloud, k=8)
    sizes = [len(ts.cloud)]
    for it in range(3):
        loss = float(ts.step(cams, targets).item())
        assert np.isfinite(loss)
        stats = ss.DensifyStats.zeros(len(ts.cloud))
        stats.accumulate(ts.grads["ss_grad"], ts.view_count)
        # the same pass on copies of the state
        ref_cloud = ss.SurfelCloud(*(getattr(ts.cloud, k).clone() for k in FIELDS))
        ref_opt = ss.Adam()
        for k in FIELDS:
            ref_opt.m[k], ref_opt.v[k], ref_opt.t[k] = ts.adam.m[k].clone(), ts.adam.v[k].clone(), ts.adam.t[k]
        want, want_map, want_reasons = ss.refine_topology(ref_cloud, stats, index.mean_dist, int(6300), quantile=0.95,
                                                          optimizer=ref_opt)
        imap, reasons = ts.refine(stats, index.mean_dist, int(6300), quantile=0.95)
        assert reasons == want_reasons and torch.equal(imap, want_map)
        for k in FIELDS:
            assert torch.equal(getattr(ts.cloud, k), getattr(want, k)), k
            assert torch.equal(ts.adam.m[k], ref_opt.m[k]) and torch.equal(ts.adam.v[k], ref_opt.v[k])
        index.rebuild(ts.cloud)
        sizes.append(len(ts.cloud))
    assert sizes[-1] != sizes[0] and max(sizes) <= 6300
