"""Adam and the refinement scan on the device vs the reference golden
fixtures (tests/golden/optim_refine.npz) and the oracle (needs a B200)."""

import numpy as np
import pytest
import torch

from golden_io import cloud_of, load
from parity import grad_close, host

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402


def test_adam_trace_matches_reference():
    d = load("optim_refine")
    p = torch.tensor(d["adam_p0"], device="cuda")
    opt = ss.Adam()
    for k in range(3):
        opt.step("x", p, torch.tensor(d["adam_grads"][k], device="cuda", dtype=torch.float32), 0.01)
        np.testing.assert_allclose(host(p), d["adam_traj"][k], rtol=2e-6, atol=2e-7)


@pytest.mark.parametrize("state", [torch.float64, torch.float32])
def test_adam_state_precision(state):
    """Moments are float64 by default like the reference (adam.py:26-28);
    float32 is an option.  Both follow the reference trace, the float64 state
    to the float32 rounding of the parameter."""
    d = load("optim_refine")
    for multi in (False, True):
        p = torch.tensor(d["adam_p0"], device="cuda")
        opt = ss.Adam(state_dtype=state)
        for k in range(3):
            g = torch.tensor(d["adam_grads"][k], device="cuda", dtype=torch.float32)
            if multi:
                opt.step_multi([("x", p, g, 0.01)])
            else:
                opt.step("x", p, g, 0.01)
            np.testing.assert_allclose(host(p), d["adam_traj"][k], rtol=2e-6, atol=2e-7)
        assert opt.m["x"].dtype == state and opt.v["x"].dtype == state
        arrays = opt.state_arrays()
        assert arrays["adam_m_x"].dtype == (np.float64 if state == torch.float64 else np.float32)
        back = ss.Adam(state_dtype=state)
        back.load_state_arrays(arrays)
        assert torch.equal(back.m["x"], opt.m["x"]) and back.t["x"] == 3


def test_adam_master_params_match_reference_update_exactly():
    """Adam(master_params=True): float64 masters stepped with the reference's
    numpy update operation by operation (adam.py:31-41) and quaternions
    renormalised in float64 (surfels.py:31-37, train.py:246) -- bit-equal to
    the oracle's float64 restatement given the same (float32) gradients; the
    kernels' float32 tensors hold the rounded masters."""
    rng = np.random.default_rng(11)
    n = 1000
    p0 = rng.normal(size=(n, 3))
    q0 = rng.normal(size=(n, 4))
    q0 /= np.linalg.norm(q0, axis=-1, keepdims=True)
    opt = ss.Adam(master_params=True)
    p = torch.tensor(p0, device="cuda", dtype=torch.float32)
    q = torch.tensor(q0, device="cuda", dtype=torch.float32)
    opt.set_master("x", p0)
    opt.set_master("q", q0)
    rp, rq = p0.copy(), q0.copy()
    mp, vp, mq, vq = (np.zeros_like(a) for a in (p0, p0, q0, q0))
    for t in range(1, 4):
        gp = rng.normal(size=p0.shape).astype(np.float32)
        gq = rng.normal(size=q0.shape).astype(np.float32)
        opt.step_multi([("x", p, torch.tensor(gp, device="cuda"), 0.01),
                        ("q", q, torch.tensor(gq, device="cuda"), 0.005)], renorm_quats="q")
        O.adam_step(rp, gp, mp, vp, t, 0.01)
        O.adam_step(rq, gq, mq, vq, t, 0.005)
        rq /= np.linalg.norm(rq, axis=-1, keepdims=True)
        assert np.array_equal(host(opt.p64["x"]), rp)
        assert np.array_equal(host(opt.p64["q"]), rq)
        assert np.array_equal(host(opt.m["x"]), mp) and np.array_equal(host(opt.v["q"]), vq)
        assert np.array_equal(host(p), rp.astype(np.float32)) and np.array_equal(host(q), rq.astype(np.float32))
    # the reference's own 3-step trace (float64 gradients, rounded to float32 here)
    d = load("optim_refine")
    opt = ss.Adam(master_params=True)
    x = torch.tensor(d["adam_p0"], device="cuda")
    for k in range(3):
        opt.step_multi([("x", x, torch.tensor(d["adam_grads"][k], device="cuda", dtype=torch.float32), 0.01)])
        np.testing.assert_allclose(host(opt.p64["x"]), d["adam_traj"][k], rtol=1e-6, atol=1e-7)


def test_adam_master_remap_keeps_survivors():
    opt = ss.Adam(master_params=True)
    p = torch.arange(12, device="cuda", dtype=torch.float32).view(4, 3)
    opt.set_master("x", p.double() + 1e-9)
    opt.step_multi([("x", p, torch.ones_like(p), 0.1)])
    before = opt.p64["x"].clone()
    new = torch.full((5, 3), 7.0, device="cuda")
    opt.remap("x", torch.tensor([2, 0, -1, 3, -1], device="cuda"), param=new)
    got = opt.p64["x"]
    assert torch.equal(got[0], before[2]) and torch.equal(got[1], before[0]) and torch.equal(got[3], before[3])
    assert torch.equal(got[2], new[2].double()) and torch.equal(got[4], new[4].double())
    assert float(opt.m["x"][2].abs().sum()) == 0.0


def test_adam_remap_semantics():
    opt = ss.Adam()
    p = torch.zeros(4, 2, device="cuda")
    opt.step("x", p, torch.ones(4, 2, device="cuda"), 0.1)
    opt.remap("x", np.array([2, -1, 0]))
    assert opt.m["x"].shape == (3, 2)
    assert float(opt.m["x"][1].abs().sum()) == 0.0
    assert float(opt.m["x"][0, 0]) == pytest.approx(0.1)


def test_refine_topology_matches_reference():
    d = load("optim_refine")
    cloud = ss.SurfelCloud.from_host(cloud_of(d))
    stats = ss.DensifyStats(torch.tensor(d["grad_sum"], device="cuda"),
                            torch.tensor(d["view_count"], device="cuda", dtype=torch.int64))
    new, index_map, reasons = ss.refine_topology(cloud, stats, d["mean_dist"], int(d["max_surfels"]), quantile=0.9)
    np.testing.assert_array_equal(host(index_map), d["index_map"])
    assert [reasons[k] for k in ("stale", "isolated", "floater", "split")] == list(d["reasons"])
    for k in ("quats", "albedo_raw", "metallic_raw", "roughness_raw"):
        np.testing.assert_array_equal(host(getattr(new, k)), d[f"new_{k}"])
    np.testing.assert_allclose(host(new.centers), d["new_centers"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(host(new.log_scales), d["new_log_scales"], rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("n", [2, 3000])
def test_isolation_matches_brute_force(n):
    rng = np.random.default_rng(n)
    c = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    c[1] = c[0]  # an exact duplicate is a neighbour at distance 0
    ls = np.log(rng.uniform(0.005, 0.05, (n, 2))).astype(np.float32)
    cloud = ss.SurfelCloud(c, np.tile([1.0, 0, 0, 0], (n, 1)), ls, np.zeros((n, 3)), np.zeros(n), np.zeros(n))
    got = host(ss.densify.isolated_mask(cloud))
    d2 = np.sum((c[:, None, :].astype(np.float64) - c[None, :, :]) ** 2, axis=2)
    np.fill_diagonal(d2, np.inf)
    want = np.sqrt(d2.min(axis=1)) > 3.0 * np.exp(ls.astype(np.float64)).max(axis=1)
    np.testing.assert_array_equal(got, want)


def test_split_children_match_oracle():
    d = load("optim_refine")
    cl = cloud_of(d)
    cloud = ss.SurfelCloud.from_host(cl)
    mask = np.zeros(len(cl.centers), bool)
    mask[[3, 10, 77, 150]] = True
    new, index_map = ss.split_cloud(cloud, mask)
    cp, cm, cls = O.split_children(cl.centers, cl.quats, cl.log_scales, np.flatnonzero(mask))
    nk = len(cl.centers) - 4
    np.testing.assert_allclose(host(new.centers)[nk:nk + 4], cp, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(host(new.centers)[nk + 4:], cm, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(host(new.log_scales)[nk:nk + 4], cls, rtol=1e-6, atol=1e-6)
    assert (host(index_map)[nk:] == -1).all()


def test_train_step_stats_feed_refinement():
    """A V-view TrainStep yields the DensifyStats of V per-view
    backward_image + accumulate calls (densify.py:35-37, train.py:250):
    grad_sum = sum_v ss_grad_v, view_count = sum_v touched_v (views, not
    pixels), so mean_grad = sum_v ss / #views touched."""
    from paper_2605_05876_b200 import scenes
    gt = scenes.config0(3, 2000)
    cams = ss.fibonacci_cameras(3, 3.0, 64, 64, fov_y_deg=40.0)
    env = ss.EnvironmentLight.from_base(scenes.env_lognormal(8, 16, 1))
    targets = [ss.render(ss.SurfelCloud(**gt), c, ss.RenderOptions(), env=env).rgb.contiguous() for c in cams]
    cloud = ss.SurfelCloud(**scenes.perturb(gt, 4))
    ts = ss.TrainStep(cloud, env, 64, 64)
    ts.gradients(cams, targets)
    stats = ss.DensifyStats.zeros(len(cloud))
    stats.accumulate(ts.grads["ss_grad"], ts.view_count)
    ref = ss.DensifyStats.zeros(len(cloud))
    for cam, tgt in zip(cams, targets):
        res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
        _, g = ss.photometric_loss(res.rgb, tgt, lambda_ssim=0.0)
        back = ss.backward_image(cloud, res, g_rgb=g)
        ref.accumulate(back.ss_grad, back.touched)
    assert torch.equal(stats.view_count, ref.view_count)
    assert int(stats.view_count.max()) == 3          # surfels seen from all three views
    assert int((stats.view_count == 2).sum()) > 0    # ... and from only some of them
    bad, err = grad_close(stats.grad_sum, ref.grad_sum)
    assert bad == 0, err
    bad, err = grad_close(stats.mean_grad(), ref.mean_grad())
    assert bad == 0, err
    new, imap, reasons = ss.refine_topology(cloud, stats, np.full(len(cloud), 0.001), 2300, quantile=0.95)
    assert len(new) <= 2300 and reasons["split"] > 0


def test_adam_multi_equals_per_tensor_steps():
    """The fused multi-tensor launch (with the quaternion renormalisation)
    equals per-tensor Adam.step + normalize_quats bit for bit."""
    rng = np.random.default_rng(9)
    shapes = {"centers": (500, 3), "quats": (500, 4), "log_scales": (500, 2), "metallic_raw": (500,)}
    ps = {k: torch.tensor(rng.normal(size=s), dtype=torch.float32, device="cuda") for k, s in shapes.items()}
    qs = {k: v.clone() for k, v in ps.items()}
    a, b = ss.Adam(), ss.Adam()
    for it in range(3):
        gs = {k: torch.tensor(rng.normal(size=s), dtype=torch.float32, device="cuda") for k, s in shapes.items()}
        for k in shapes:
            a.step(k, ps[k], gs[k], 0.01 * (it + 1))
        ss.normalize_quats(ps["quats"])
        b.step_multi([(k, qs[k], gs[k], 0.01 * (it + 1)) for k in shapes], renorm_quats="quats")
    for k in shapes:
        assert torch.equal(ps[k], qs[k]), k
        assert torch.equal(a.m[k], b.m[k]) and torch.equal(a.v[k], b.v[k])
