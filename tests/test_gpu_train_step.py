"""The fused training-step path (ss_train_forward / ss_train_backward) against
the API path and the oracle on the same seeded inputs (needs a B200)."""

import numpy as np
import pytest
import torch

from types import SimpleNamespace

from parity import grad_close, grad_outliers, host

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import PARAMS, TrainStep  # noqa: E402


def _scene(n=3000, res=96, seed=0):
    gt = scenes.config0(seed, n)
    init = scenes.perturb(gt, seed + 1)
    env_base = scenes.env_lognormal(16, 32, seed + 2)
    cams = ss.fibonacci_cameras(4, 3.0, res, res, fov_y_deg=40.0)
    gt_env = ss.EnvironmentLight.from_base(env_base)
    gtc = ss.SurfelCloud(**gt)
    targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
    return init, env_base, cams, targets


def _oracle_step(init, env_base, cams, targets, images):
    """Sum over views of the ORACLE's render -> L1 -> backward_image (the
    reference algorithm, not a CUDA path), with the L1 sign pattern of the
    step's own fused-forward images (`images`, TrainStep.captured_rgb): the
    step shades in float32, so residuals below ~1e-7 may flip sign vs the
    oracle's float64 image."""
    co = SimpleNamespace(**init)
    oenv = O.EnvOracle(np.log(np.asarray(env_base, np.float64)))
    acc, views = None, np.zeros(len(init["centers"]), np.float32)
    for cam, tgt, img in zip(cams, targets, images):
        ores = O.render(co, cam, env=oenv)
        rgb = host(img).astype(np.float64)
        g = np.sign(rgb - host(tgt)) / rgb.size
        og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
        views += og["touched"]
        if acc is None:
            acc = {k: np.array(og[k], np.float64) for k in list(PARAMS) + ["ss_grad", "env_base_log"]}
        else:
            for k in acc:
                acc[k] += og[k]
    acc["view_count"] = views
    return acc


def _assert_step_matches_oracle(ts, ref):
    bad = {}
    for k in list(PARAMS) + ["ss_grad"]:
        outl, n = grad_outliers(ts.grads[k], ref[k].reshape(ts.grads[k].shape))
        if n:
            bad[k] = (n, outl)
    outl, n = grad_outliers(ts.g_env_log, ref["env_base_log"])
    if n:
        bad["env_base_log"] = (n, outl)
    assert not bad, bad
    np.testing.assert_array_equal(host(ts.view_count), ref["view_count"])


def test_train_step_gradients_match_oracle():
    """The fused multi-view step vs the oracle summed over the same views."""
    init, env_base, cams, targets = _scene()
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, 96, 96)
    ts.captured_rgb = []
    ts.gradients(cams, targets)
    _assert_step_matches_oracle(ts, _oracle_step(init, env_base, cams, targets, ts.captured_rgb[-len(cams):]))


def test_train_step_gradients_match_api_path():
    init, env_base, cams, targets = _scene()
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, 96, 96)
    ts.gradients(cams, targets)
    torch.cuda.synchronize()
    # API path: render -> L1 -> backward_image, summed over views
    acc = {k: torch.zeros_like(ts.grads[k]) for k in PARAMS}
    loss = 0.0
    d_diff = torch.zeros(env.base.shape, device="cuda", dtype=torch.float64)
    d_spec = torch.zeros(env.specular.shape, device="cuda", dtype=torch.float64)
    for cam, tgt in zip(cams, targets):
        res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
        val, g = ss.photometric_loss(res.rgb, tgt, lambda_ssim=0.0)
        loss += val * res.rgb.numel()
        back = ss.backward_image(cloud, res, g_rgb=g, path="walk")  # not the record kernel the step runs
        for k in PARAMS:
            acc[k] += getattr(back, k).reshape(acc[k].shape)
        d_diff += back.d_diffuse
        d_spec += back.d_specular
    assert float(ts.loss_f.item()) == pytest.approx(loss, rel=1e-5)
    for k in PARAMS:
        bad, err = grad_close(ts.grads[k], acc[k])
        assert bad == 0, (k, err)
    _, g_env = env.env_gradient(d_diff, d_spec)
    assert grad_close(ts.g_env_log, g_env, rel=1e-3)[0] == 0


def test_train_step_reduces_loss():
    init, env_base, cams, targets = _scene(n=2000, res=64)
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, 64, 64, lrs={"centers": 1e-3, "quats": 1e-3, "log_scales": 5e-3,
                                             "albedo_raw": 2e-2, "metallic_raw": 2e-2, "roughness_raw": 2e-2,
                                             "env_base_log": 1e-2})
    first = float(ts.step(cams, targets).item())
    for _ in range(30):
        last = float(ts.step(cams, targets).item())
    assert last < 0.9 * first
    assert torch.isfinite(cloud.centers).all()
    q = cloud.quats
    assert torch.allclose(q.norm(dim=1), torch.ones(len(cloud), device=q.device), atol=1e-5)


def test_host_targets_path_equals_resident():
    init, env_base, cams, targets = _scene(n=1500, res=64)
    outs = []
    for host_mode in (False, True):
        cloud = ss.SurfelCloud(**init)
        env = ss.EnvironmentLight.from_base(env_base)
        ts = TrainStep(cloud, env, 64, 64)
        if host_mode:
            loss = ts.step_host(cams, [t.cpu().pin_memory() for t in targets])
        else:
            loss = ts.step(cams, targets)
        outs.append((float(loss.item()), cloud.centers.clone()))
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("with_masks,cons", [(False, 0.0), (True, 0.0), (True, 2e-4)])
def test_photometric_train_step_matches_api_path(with_masks, cons):
    """loss="photometric" (the reference fit loss, train.py:194-213: hdr-loss
    tone map, 0.8 L1 + 0.2 (1 - SSIM), + lambda_sil silhouette, + the
    consolidation penalty of the main phase) through the deferred-loss
    kernels vs render -> image_loss / silhouette_loss -> backward_image
    (walk path) summed over views."""
    init, env_base, cams, targets = _scene(n=2500, res=80)
    rng = np.random.default_rng(5)
    masks = [torch.as_tensor((rng.uniform(size=(80, 80)) > 0.5).astype(np.float32), device="cuda")
             for _ in cams] if with_masks else None
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, 80, 80, loss="photometric", lambda_sil=0.3, cons_scale=cons)
    ts.gradients(cams, targets, masks)
    torch.cuda.synchronize()
    acc = {k: torch.zeros_like(ts.grads[k]) for k in PARAMS}
    loss = cons_total = 0.0
    d_diff = torch.zeros(env.base.shape, device="cuda", dtype=torch.float64)
    d_spec = torch.zeros(env.specular.shape, device="cuda", dtype=torch.float64)
    for i, (cam, tgt) in enumerate(zip(cams, targets)):
        res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
        val, g = ss.image_loss(res.rgb, tgt, tone="hdr-loss", lambda_ssim=0.2)
        loss += val
        g_alpha = None
        if with_masks:
            sv, ga = ss.silhouette_loss(res.alpha, masks[i])
            loss += 0.3 * sv
            g_alpha = 0.3 * ga
        back = ss.backward_image(cloud, res, g_rgb=g, g_alpha=g_alpha, cons_scale=cons, path="walk")
        loss += back.cons_loss
        cons_total += back.cons_loss
        for k in PARAMS:
            acc[k] += getattr(back, k).reshape(acc[k].shape)
        d_diff += back.d_diffuse
        d_spec += back.d_specular
    assert float(ts.loss_f.item()) == pytest.approx(loss, rel=1e-5)
    assert (cons_total > 0.01 * loss) == (cons > 0.0)  # the penalty is exercised when on
    for k in PARAMS:
        bad, err = grad_close(ts.grads[k], acc[k])
        assert bad == 0, (k, err)
    _, g_env = env.env_gradient(d_diff, d_spec)
    assert grad_close(ts.g_env_log, g_env, rel=1e-3)[0] == 0


@pytest.mark.parametrize("wh", [(97, 61), (33, 120)])
def test_train_step_ragged_image(wh):
    """Image sizes that are not tile multiples (partial tiles and 8x4 warp
    blocks at the right/bottom edges), training path vs API path."""
    W, H = wh
    gt = scenes.config0(2, 2000)
    init = scenes.perturb(gt, 3)
    env_base = scenes.env_lognormal(16, 32, 4)
    cams = ss.fibonacci_cameras(3, 3.0, W, H, fov_y_deg=40.0)
    gt_env = ss.EnvironmentLight.from_base(env_base)
    gtc = ss.SurfelCloud(**gt)
    targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, W, H)
    ts.captured_rgb = []
    ts.gradients(cams, targets)
    torch.cuda.synchronize()
    acc = {k: torch.zeros_like(ts.grads[k]) for k in PARAMS}
    for cam, tgt in zip(cams, targets):
        res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
        _, g = ss.photometric_loss(res.rgb, tgt, lambda_ssim=0.0)
        back = ss.backward_image(cloud, res, g_rgb=g, path="walk")
        for k in PARAMS:
            acc[k] += getattr(back, k).reshape(acc[k].shape)
    for k in PARAMS:
        bad, err = grad_close(ts.grads[k], acc[k])
        assert bad == 0, (k, err)
    _assert_step_matches_oracle(ts, _oracle_step(init, env_base, cams, targets, ts.captured_rgb[-len(cams):]))


def test_train_step_with_normal_consistency():
    """set_normal_consistency adds lambda_nc * normal_consistency_loss (value and
    quaternion gradient, train.py:216-221) once per view of the step: a
    V-view step equals the sum of V reference steps."""
    init, env_base, cams, targets = _scene(n=2000, res=64)
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, 64, 64)
    ts.gradients(cams, targets)
    base_loss = float(ts.loss_f.item())
    base_q = ts.grads["quats"].clone()
    idx = ss.NeighborIndex(cloud, k=8)
    ts.set_normal_consistency(idx, 0.05)
    ts.gradients(cams, targets)
    nc, g = ss.normal_consistency_loss(cloud, idx)
    V = len(cams)
    assert float(ts.loss_f.item()) == pytest.approx(base_loss + 0.05 * V * nc, rel=1e-6)
    bad, err = grad_close(ts.grads["quats"], base_q + 0.05 * V * g.reshape(base_q.shape))
    assert bad == 0, err
    ts.set_normal_consistency(None, 0.0)
    ts.gradients(cams, targets)
    assert float(ts.loss_f.item()) == pytest.approx(base_loss, rel=1e-6)


def test_step_host_includes_normal_consistency():
    """The pinned-host entry point (the bench's e2e path) applies the same
    step as step(), normal-consistency term included."""
    init, env_base, cams, targets = _scene(n=1500, res=64)
    outs = []
    for host_mode in (False, True):
        cloud = ss.SurfelCloud(**init)
        env = ss.EnvironmentLight.from_base(env_base)
        ts = TrainStep(cloud, env, 64, 64)
        ts.set_normal_consistency(ss.NeighborIndex(cloud, k=8), 0.05)
        if host_mode:
            loss = ts.step_host(cams, [t.cpu().pin_memory() for t in targets])
        else:
            loss = ts.step(cams, targets)
        outs.append((float(loss.item()), cloud.quats.clone()))
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1])


def test_pair_overflow_grows_and_reruns():
    """A step whose views need more pairs than the buffers hold grows them
    and re-runs the views before Adam: the parameters after the step equal
    those of a step with ample buffers (no truncated tile list reaches the
    optimiser; the offsets are clamped, so nothing reads out of bounds)."""
    init, env_base, cams, targets = _scene(n=1500, res=64)
    outs = []
    for cap in (None, 300):
        cloud = ss.SurfelCloud(**init)
        env = ss.EnvironmentLight.from_base(env_base)
        ts = TrainStep(cloud, env, 64, 64, pair_capacity=cap)
        loss = float(ts.step(cams, targets).item())
        outs.append((loss, cloud.centers.clone(), ts.regrows, ts.capacity))
    assert outs[1][2] == 1 and outs[1][3] > 300
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1])


def test_nonfinite_colour_raises_in_step():
    init, env_base, cams, targets = _scene(n=500, res=32)
    bad = dict(init)
    bad["albedo_raw"] = bad["albedo_raw"].copy()
    bad["metallic_raw"] = bad["metallic_raw"].copy()
    bad["metallic_raw"][7] = np.nan
    cloud = ss.SurfelCloud(**bad)
    env = ss.EnvironmentLight.from_base(env_base)
    ts = TrainStep(cloud, env, 32, 32)
    with pytest.raises(ValueError):
        ts.step(cams, [torch.zeros(32, 32, 3, device="cuda")] * len(cams))


def test_graph_replay_matches_eager():
    """TrainStep.step(graph=True): the captured gradient pass replays the
    eager one (same gradients up to the float atomics' order), the cache is
    keyed by the cameras, and a pair-buffer overflow drops it and re-runs."""
    gt = scenes.config0(0, 10_000)
    cams = ss.fibonacci_cameras(4, 3.0, 128, 128)
    env = ss.EnvironmentLight(np.log(scenes.env_lognormal(16, 32, 2)))
    targets = [ss.render(ss.SurfelCloud(**gt), c, ss.RenderOptions(), env=env).rgb.contiguous() for c in cams]
    cloud = ss.SurfelCloud(**scenes.perturb(gt, 1))
    ts = TrainStep(cloud, env, 128, 128, streams=2)
    ts.gradients(cams, targets)
    ref = {k: ts.grads[k].clone() for k in PARAMS}
    ref_env = ts.g_env_log.clone()
    for _ in range(3):  # eager + capture, then two replays
        ts.gradients_graphed(cams, targets)
        for k in PARAMS:
            torch.testing.assert_close(ts.grads[k], ref[k], rtol=1e-5, atol=1e-6 * float(ref[k].abs().max()))
        torch.testing.assert_close(ts.g_env_log, ref_env, rtol=1e-5, atol=1e-6 * float(ref_env.abs().max()))
    assert len(ts._graphs) == 1
    ts.gradients_graphed(cams[:2], targets[:2])  # another camera list: its own graph
    assert len(ts._graphs) == 2
    # replay overflow: the surfels grow in place (as Adam would grow them),
    # the captured pass overflows its pair buffers, which grow, and the step
    # re-runs eagerly (and drops the stale graphs)
    ts._alloc_pairs(int(ts.bufs[0].offsets[-1].item()) + 64)
    ts._graphs.clear()
    ts.gradients_graphed(cams[:1], targets[:1])
    ts.gradients_graphed(cams[:1], targets[:1])
    grows = ts.regrows
    with torch.no_grad():
        cloud.log_scales.add_(0.4)
    ts.gradients_graphed(cams[:1], targets[:1])
    assert ts.regrows > grows and len(ts._graphs) == 0
    want = {k: ts.grads[k].clone() for k in PARAMS}
    ts.gradients(cams[:1], targets[:1])
    for k in PARAMS:
        torch.testing.assert_close(want[k], ts.grads[k], rtol=1e-5, atol=1e-6 * float(ts.grads[k].abs().max()))


def test_diffuse_taps_per_step_equal_per_view():
    """ss_chain_backward_prepared + ss_diffuse_scatter (the normal's diffuse
    lookup from the step prepass, its bilinear taps applied once per step) vs
    the per-view scatter of ss_chain_backward: the same derived-map gradient
    and parameter gradients up to float summation order."""
    init, env_base, cams, targets = _scene()
    out = {}
    for per_step in (True, False):
        ts = TrainStep(ss.SurfelCloud(**init), ss.EnvironmentLight.from_base(env_base), 96, 96, streams=1)
        if not per_step:
            ts._diffuse_per_step = lambda: False
        ts.gradients(cams, targets)
        torch.cuda.synchronize()
        out[per_step] = ({k: ts.grads[k].clone() for k in PARAMS}, ts.d_diffuse.clone(), ts.g_env_log.clone())
    (ga, da, ea), (gb, db, eb) = out[True], out[False]
    assert float(da.abs().max()) > 0
    # the float32 per-view maps vs the float32 per-surfel view sums: texels whose
    # contributions cancel differ beyond 1e-5 of themselves, so the bar is the
    # gradient tolerance of every parity test (rel 1e-3, floor 1e-5 x max)
    assert grad_close(da, db)[0] == 0, grad_outliers(da, db)
    assert grad_close(ea, eb)[0] == 0, grad_outliers(ea, eb)
    for k in PARAMS:
        assert grad_close(ga[k], gb[k])[0] == 0, (k, grad_outliers(ga[k], gb[k]))
    # and far inside it in aggregate
    assert float((da - db).abs().max()) <= 1e-4 * float(db.abs().max())
