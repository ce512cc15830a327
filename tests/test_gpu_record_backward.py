"""The record-parallel backward of the training step (csrc/train_step.cu:
area-class sort, 8-lane groups, medium and huge big-rect paths) against the
walk-based backward that mirrors the reference (_backward_kernel,
backward.py:48-321; both are checked against the reference goldens in
test_gpu_parity.py), with and without the consolidation penalty.  Needs a
B200."""

import numpy as np
import pytest
import torch

from parity import grad_close, host

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw", "ss_grad")


def _mixed_cloud(n=600, seed=0, big=20, huge=5):
    """Surfels on the unit sphere: most small, `big` with rects of a few
    thousand pixels (medium path), `huge` with rects above 8192 px."""
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(n, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    ls = rng.uniform(np.log(0.008), np.log(0.03), size=(n, 2))
    ls[:big] = np.log(rng.uniform(0.04, 0.08, size=(big, 2)))
    ls[big:big + huge] = np.log(rng.uniform(0.15, 0.3, size=(huge, 2)))
    return scenes._raw_cloud(p, p, ls, rng.uniform(0, 1, (n, 3)), rng.uniform(0.1, 0.9, n), rng.uniform(0, 1, n))


def _both_paths(cloud, cam, env, g_seed=1, cons_scale=0.0):
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    g = torch.from_numpy(np.random.default_rng(g_seed).normal(0, 1e-3, (cam.height, cam.width, 3)).astype(np.float32))
    g = g.cuda()
    rec = ss.backward_image(cloud, res, g_rgb=g, cons_scale=cons_scale, path="records")
    walk = ss.backward_image(cloud, res, g_rgb=g, cons_scale=cons_scale, path="walk")
    return res, rec, walk


def _rect_areas(res):
    st = res.state
    keep = st.cull == 0
    r = st.records[keep][:, 20:24].contiguous().view(torch.int32).long()
    return host((r[:, 2] - r[:, 0]) * (r[:, 3] - r[:, 1]))


@pytest.mark.parametrize("wh,cons", [((200, 200), 0.0), ((231, 157), 0.0), ((200, 200), 1e-3), ((231, 157), 1e-2)])
def test_record_backward_matches_walk_with_big_rects(wh, cons):
    W, H = wh
    cloud = ss.SurfelCloud(**_mixed_cloud())
    env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 2))
    cam = ss.fibonacci_cameras(3, 3.0, W, H, fov_y_deg=40.0)[1]
    res, rec, walk = _both_paths(cloud, cam, env, cons_scale=cons)
    assert rec.cons_loss == pytest.approx(walk.cons_loss, rel=1e-5, abs=1e-12)
    if cons > 0.0:
        assert rec.cons_loss > 0.0
    a = _rect_areas(res)
    assert (a > 512).sum() >= 2 and (a > 8192).sum() >= 1, "scene must exercise the medium and huge paths"
    np.testing.assert_array_equal(host(rec.touch_count), host(walk.touch_count))
    for k in KEYS:
        bad, err = grad_close(getattr(rec, k), getattr(walk, k))
        assert bad == 0, (k, err)
    assert grad_close(rec.env_base_log, walk.env_base_log)[0] == 0


def test_record_backward_single_area_class():
    """Every record in one area class (equal scales, flat facing plane):
    the class sort degenerates to one bucket."""
    n = 24 * 24
    g = np.stack(np.meshgrid(np.linspace(-0.6, 0.6, 24), np.linspace(-0.6, 0.6, 24)), -1).reshape(-1, 2)
    centers = np.concatenate([g, np.zeros((n, 1))], 1)
    normals = np.tile([0.0, 0.0, 1.0], (n, 1))
    ls = np.full((n, 2), np.log(0.02))
    rng = np.random.default_rng(5)
    cloud = ss.SurfelCloud(**scenes._raw_cloud(centers, normals, ls, rng.uniform(0, 1, (n, 3)),
                                               rng.uniform(0.1, 0.9, n), rng.uniform(0, 1, n)))
    cam = ss.Camera.perspective(96, 96, 40.0, eye=(0.0, 0.0, 2.5), target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0))
    env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 3))
    res, rec, walk = _both_paths(cloud, cam, env, g_seed=7)
    a = _rect_areas(res)
    assert a.size > 0 and len(np.unique(a)) <= 4
    np.testing.assert_array_equal(host(rec.touch_count), host(walk.touch_count))
    for k in KEYS:
        bad, err = grad_close(getattr(rec, k), getattr(walk, k))
        assert bad == 0, (k, err)


def test_record_backward_with_consolidation_at_config2_size():
    """BASELINE config-2 view (1M surfels, 800x800) with the reference's
    main-phase consolidation weight: record path vs walk path."""
    gt = scenes.config2(0, 1_000_000)
    cloud = ss.SurfelCloud(**scenes.perturb(gt, 1))
    env = ss.EnvironmentLight(np.log(scenes.env_lognormal(128, 256, 2)))
    cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[21]
    res, rec, walk = _both_paths(cloud, cam, env, g_seed=4, cons_scale=100.0 / (800 * 800))
    assert rec.cons_loss > 0.0
    assert rec.cons_loss == pytest.approx(walk.cons_loss, rel=1e-5)
    np.testing.assert_array_equal(host(rec.touch_count), host(walk.touch_count))
    for k in KEYS:
        bad, err = grad_close(getattr(rec, k), getattr(walk, k))
        assert bad <= 1e-4 * getattr(rec, k).numel(), (k, bad, err)
