"""Parity at BASELINE sizes (needs a B200 and a multi-core host for the oracle).

Config 2 (1M surfels, 800x800, env 128x256): one view, full pipeline on both
sides -- tile lists and sort order bit-exact, images within 1e-4, training
gradients (fused path) within the gradient tolerance.  Config 3 (16
concentric shells, k_max stop): layer counts and the discard statistic exact.
Config 0 (10k surfels, 128x128): the whole training step vs the oracle.
"""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from parity import grad_close, grad_outliers, host, image_close

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import PARAMS, TrainStep  # noqa: E402


def _oracle_env(base_log, levels=6):
    return O.EnvOracle(np.asarray(base_log, np.float64), levels=levels)


def _check_step_grads(ts, og, label, ores=None, floor=1e-5):
    """Every parameter channel, ss_grad and the env gradient of a training
    step vs the oracle's backward_image: 0 entries outside the gradient
    tolerance (north_star: 1e-3 relative, with the 1e-5 x array-scale floor
    of tests/parity.py); outliers are listed with their magnitudes.  The
    per-view touched flags equal the step's view counts (1 view)."""
    report = {}
    if ores is not None:  # the step's float32-shaded image vs the oracle's float64 one
        bad, err = image_close(ts.captured_rgb[-1], ores.rgb)
        assert bad == 0, (label, "fused-forward image", bad, err)
    pairs = [(k, ts.grads[k], og[k]) for k in PARAMS]
    pairs += [("ss_grad", ts.grads["ss_grad"], og["ss_grad"]), ("env_base_log", ts.g_env_log, og["env_base_log"])]
    for k, got, ref in pairs:
        outl, nbad = grad_outliers(got, ref, floor=floor)
        if nbad:
            report[k] = (nbad, outl)
    assert not report, f"{label}: gradient entries outside tolerance: {report}"
    np.testing.assert_array_equal(host(ts.view_count), og["touched"].astype(np.float32))


@pytest.fixture(scope="module")
def config2():
    gt = scenes.config2(0, 1_000_000)
    opt = scenes.perturb(gt, 1)
    base_log = np.log(scenes.env_lognormal(128, 256, 2))
    cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[5]
    return gt, opt, base_log, cam


def test_config2_forward_full_size(config2):
    gt, opt, base_log, cam = config2
    cloud = ss.SurfelCloud(**opt)
    env = ss.EnvironmentLight(base_log)
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    oenv = _oracle_env(base_log)
    ores = O.render(SimpleNamespace(**opt), cam, env=oenv)
    np.testing.assert_array_equal(host(res.tile_offsets), ores.tile_offsets)
    np.testing.assert_array_equal(host(res.pair_rec), ores.pair_rec)
    np.testing.assert_array_equal(host(res.nlayers), ores.nlayers)
    for k in ("rgb", "alpha", "depth"):
        bad, err = image_close(getattr(res, k), getattr(ores, k))
        assert bad == 0, (k, bad, err)
    # the layer-count histogram is a size-independent summary of grouping parity
    assert res.stats["pairs"] == len(ores.pair_rec) and res.stats["discarded_overflow"] == ores.discarded


def test_config2_training_gradients_full_size(config2):
    gt, opt, base_log, cam = config2
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    ts = TrainStep(cloud, env, 800, 800)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    val, _ = O.photometric_l1(ores.rgb, host(target))
    assert float(ts.loss_f.item()) / (800 * 800 * 3) == pytest.approx(val, rel=1e-4)
    # L1's sign(rgb - target) is discontinuous: pixels whose residual is below
    # the rounding of the image (the step shades in float32, the oracle in
    # float64: colours differ by ~1e-7 relative) can flip sign between the
    # two implementations, and one flipped pixel moves every gradient of the
    # few surfels covering it.  Feed the oracle the sign pattern of the
    # step's own fused-forward image so the comparison isolates the backward.
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)  # the step's own image (float32 shading)
    g = np.sign(rgb - host(target)) / rgb.size
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    _check_step_grads(ts, og, "config2", ores)


def test_config3_kmax_stress():
    cl = scenes.config3(0, 120_000)
    cam = ss.fibonacci_cameras(16, 3.5, 512, 512)[3]
    colors = np.random.default_rng(1).uniform(0, 1, (len(cl["centers"]), 3))
    res = ss.render(ss.SurfelCloud(**cl), cam, ss.RenderOptions(), colors=colors)
    ores = O.render(SimpleNamespace(**cl), cam, colors=colors)
    np.testing.assert_array_equal(host(res.pair_rec), ores.pair_rec)
    np.testing.assert_array_equal(host(res.nlayers), ores.nlayers)
    assert int(host(res.nlayers).max()) == 16
    assert res.stats["discarded_overflow"] == ores.discarded > 0
    bad, err = image_close(res.rgb, ores.rgb)
    assert bad == 0, err


def test_config3_training_backward_kmax():
    """The walk-free training backward reproduces the k_max stop: gradients
    vs the ORACLE's backward_image (not the CUDA API path)."""
    cl = scenes.config3(2, 60_000)
    cam = ss.fibonacci_cameras(16, 3.5, 256, 256)[1]
    base_log = np.log(scenes.env_lognormal(16, 32, 3))
    env = ss.EnvironmentLight(base_log)
    rng = np.random.default_rng(4)
    target = torch.tensor(rng.uniform(0, 1, (256, 256, 3)), device="cuda", dtype=torch.float32)
    cloud = ss.SurfelCloud(**cl)
    ts = TrainStep(cloud, env, 256, 256)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**cl)
    ores = O.render(co, cam, env=oenv)
    assert ores.discarded > 0 and int(ores.nlayers.max()) == 16
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)  # the step's own image (float32 shading)
    g = np.sign(rgb - host(target)) / rgb.size
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    _check_step_grads(ts, og, "config3-small")


def test_config3_full_size_vs_oracle():
    """BASELINE config 3 at full size: 500k surfels on 16 concentric shells,
    1024x1024, env 64x128 -- tile lists and sort order bit-exact, layer
    counts (k_max = 16 stop) and the discarded-record statistic exact,
    images within 1e-4, training gradients vs the oracle
    (rasterizer.py:168-196, backward.py:86-320)."""
    cl = scenes.config3(0, 500_000)
    base_log = np.log(scenes.env_lognormal(64, 128, 3))
    cam = ss.fibonacci_cameras(16, 3.5, 1024, 1024)[3]
    env = ss.EnvironmentLight(base_log)
    gt_cloud = ss.SurfelCloud(**cl)
    opt = scenes.perturb(cl, 1)
    target = ss.render(gt_cloud, cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    np.testing.assert_array_equal(host(res.tile_offsets), ores.tile_offsets)
    np.testing.assert_array_equal(host(res.pair_rec), ores.pair_rec)
    np.testing.assert_array_equal(host(res.nlayers), ores.nlayers)
    assert int(ores.nlayers.max()) == 16 and ores.discarded > 1_000_000
    assert res.stats["discarded_overflow"] == ores.discarded
    for k in ("rgb", "alpha", "depth"):
        bad, err = image_close(getattr(res, k), getattr(ores, k))
        assert bad == 0, (k, bad, err)
    ts = TrainStep(cloud, env, 1024, 1024)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)  # the step's own image (float32 shading)
    g = np.sign(rgb - host(target)) / rgb.size
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    _check_step_grads(ts, og, "config3", ores)


def test_config0_step_full_size():
    gt = scenes.config0(0, 10_000)
    opt = scenes.perturb(gt, 1)
    base_log = np.log(scenes.env_lognormal(16, 32, 2))
    cam = ss.Camera.perspective(128, 128, 40.0, (3.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    ts = TrainStep(cloud, env, 128, 128)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)  # the step's own image (float32 shading)
    g = np.sign(rgb - host(target)) / rgb.size  # same L1 sign pattern on both sides
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    _check_step_grads(ts, og, "config0", ores)


def test_config1_training_gradients_full_size():
    """Config 1 (200k surfels on a displaced torus + sphere, 512x512, env
    64x128): tile lists bit-exact, image within 1e-4, training gradients vs the
    oracle."""
    gt = scenes.config1(0, 200_000)
    opt = scenes.perturb(gt, 1)
    base_log = np.log(scenes.env_lognormal(64, 128, 3))
    cam = ss.fibonacci_cameras(8, 3.5, 512, 512)[2]
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    np.testing.assert_array_equal(host(res.pair_rec), ores.pair_rec)
    np.testing.assert_array_equal(host(res.nlayers), ores.nlayers)
    bad, err = image_close(res.rgb, ores.rgb)
    assert bad == 0, err
    ts = TrainStep(cloud, env, 512, 512)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)  # the step's own image (float32 shading)
    g = np.sign(rgb - host(target)) / rgb.size  # same L1 sign pattern on both sides
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    _check_step_grads(ts, og, "config1", ores)


def test_config4_view_full_size_vs_oracle():
    """BASELINE config 4's single view at full size: 4M surfels on the
    5-octave displaced icosphere (amplitude 0.12), 1920x1080, env 256x512 --
    tile lists, layer counts and images vs the oracle, training gradients
    (0 entries outside tolerance) and the refinement pass that follows
    every config-4 step (q = 0.95) vs the oracle's refine_topology."""
    from paper_2605_05876_b200 import densify
    gt = scenes.config2(0, 4_000_000, amp=0.12, octaves=5)
    opt = scenes.perturb(gt, 1)
    base_log = np.log(scenes.env_lognormal(256, 512, 2))
    cam = ss.fibonacci_cameras(128, 3.5, 1920, 1080)[7]
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    np.testing.assert_array_equal(host(res.tile_offsets), ores.tile_offsets)
    np.testing.assert_array_equal(host(res.pair_rec), ores.pair_rec)
    np.testing.assert_array_equal(host(res.nlayers), ores.nlayers)
    bad, err = image_close(res.rgb, ores.rgb)
    assert bad == 0, err
    ts = TrainStep(cloud, env, 1920, 1080)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)
    g = np.sign(rgb - host(target)) / rgb.size
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    _check_step_grads(ts, og, "config4", ores)
    # the per-step refinement (q = 0.95, budget 1.05 N) on this step's stats
    stats = ss.DensifyStats.zeros(len(cloud))
    stats.accumulate(ts.grads["ss_grad"], ts.view_count)
    mnd = ss.NeighborIndex(cloud, k=8).mean_dist
    new, imap, reasons = ss.refine_topology(cloud, stats, mnd, 4_200_000, quantile=0.95)
    keep, split_rows, want_map, want = O.refine_topology(
        opt["centers"], opt["quats"], opt["log_scales"], host(stats.grad_sum), host(stats.view_count), host(mnd),
        4_200_000, quantile=0.95)
    assert {k: reasons[k] for k in ("stale", "isolated", "floater", "split")} == \
        {k: want[k] for k in ("stale", "isolated", "floater", "split")}
    assert densify.LAST_REFINE["threshold"] == want["threshold"]
    np.testing.assert_array_equal(host(imap), want_map)


@pytest.mark.parametrize("cons", [0.0, 100.0 / (800 * 800)])
def test_config2_photometric_step_full_size(config2, cons):
    """The reference fit loss at config-2 size (train.py:194-213): hdr-loss
    tone map, 0.8 L1 + 0.2 (1 - SSIM 11x11), and in the main phase the depth
    consolidation penalty (lambda_cons 100 / (extent * npix)) -- the
    deferred-loss kernels vs the oracle's losses and backward_image, with the
    step's own image fed to the oracle's loss (L1 sign pattern)."""
    gt, opt, base_log, cam = config2
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    ts = TrainStep(cloud, env, 800, 800, loss="photometric", cons_scale=cons)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    rgb = host(ts.captured_rgb[-1]).astype(np.float64)
    tgt = host(target).astype(np.float64)
    val, g_map = O.photometric_loss(O.tone_map(rgb, "hdr-loss"), O.tone_map(tgt, "hdr-loss"), 0.2)
    g = O.tone_map_backward(rgb, "hdr-loss", g_map)
    oenv = _oracle_env(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    og = O.backward_image(co, ores, g, None, cons, env=oenv)
    assert float(ts.loss_f.item()) == pytest.approx(val + og["cons_loss"], rel=1e-5)
    # floor 1e-4 x array max (1e-5 elsewhere): the SSIM gradient alternates in
    # sign from pixel to pixel, so a surfel's channel sums can cancel ~1000x,
    # and the step carries its layer state (weights W, mean colours) from the
    # float32-weight forward while the reference backward re-derives it with
    # float64 weights (backward.py:160-200).  Measured at this size: 2 of 2M
    # log_scales entries (one translucent surfel, n_f = 0.005) at 2-4e-5 x max,
    # unchanged by float64 record arithmetic (parity)
    _check_step_grads(ts, og, f"config2-photometric-cons{cons > 0}", ores, floor=1e-4)
