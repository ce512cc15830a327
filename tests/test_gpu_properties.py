"""Size-independent properties of the CUDA path (SURVEY §4 "coverage gaps",
§8c): partition of unity on a surfel lattice (SPEC criterion the reference
suite leaves untested), linearity of the backward in its upstream gradient
and zero upstream -> zero gradients at the BASELINE config-2 size (1M
surfels, 800x800).  Needs a B200."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from parity import grad_close, host, image_close

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw", "ss_grad")
LINEAR = KEYS[:-1]  # ss_grad sums norms of the screen-space gradient: not linear


def _lattice(n=48, h=0.05):
    """n x n surfels on the z = 0 plane, spacing h = their scale, facing +z."""
    g = (np.arange(n) - (n - 1) / 2.0) * h
    X, Y = np.meshgrid(g, g)
    m = n * n
    centers = np.stack([X.ravel(), Y.ravel(), np.zeros(m)], 1)
    normals = np.tile([0.0, 0.0, 1.0], (m, 1))
    ls = np.full((m, 2), np.log(h))
    return scenes._raw_cloud(centers, normals, ls, np.full((m, 3), 0.5), np.full(m, 0.5), np.full(m, 0.5))


@pytest.mark.parametrize("mip", [False, True])
def test_partition_of_unity_on_a_lattice(mip):
    """Unit-spaced Gaussians (spacing = scale) sum to 2 pi (Poisson summation)
    less the rho < 3 truncation (1 - e^-4.5): interior layer weights ~6.21,
    alpha = 1 - e^-W >= 0.9979, one layer -- and the same stacks as the oracle."""
    raw = _lattice()
    cloud = ss.SurfelCloud(**raw)
    cam = ss.Camera.perspective(64, 64, 40.0, eye=(0.0, 0.0, 2.2), target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0))
    colors = np.full((len(raw["centers"]), 3), 0.25, np.float32)
    opt = ss.RenderOptions(collect_stacks=True, mip_enabled=mip)
    res = ss.render(cloud, cam, opt, colors=colors)
    w = host(res.stacks["weight_sum"])[..., 0].astype(np.float64)
    inner = w[8:-8, 8:-8]
    expect = 2.0 * np.pi * (1.0 - np.exp(-4.5))
    assert np.all(np.abs(inner / expect - 1.0) < 0.01), (inner.min(), inner.max(), expect)
    assert np.all(host(res.nlayers)[8:-8, 8:-8] == 1)
    assert float(host(res.alpha)[8:-8, 8:-8].min()) >= 0.9979
    ores = O.render(SimpleNamespace(**raw), cam, colors=colors, mip_enabled=mip, collect_stacks=True)
    bad, err = image_close(res.stacks["weight_sum"], ores.stacks["weight_sum"], rel=1e-4, abs_=1e-6)
    assert bad == 0, err
    np.testing.assert_array_equal(host(res.nlayers), ores.nlayers)


@pytest.fixture(scope="module")
def config2_view():
    gt = scenes.config2(0, 1_000_000)
    cloud = ss.SurfelCloud(**scenes.perturb(gt, 1))
    env = ss.EnvironmentLight(np.log(scenes.env_lognormal(128, 256, 2)))
    cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[9]
    return cloud, env, ss.render(cloud, cam, ss.RenderOptions(), env=env)


def _grads(cloud, res, g):
    b = ss.backward_image(cloud, res, g_rgb=g)
    return {k: getattr(b, k).double() for k in KEYS}, b


def test_backward_is_linear_in_the_upstream_gradient(config2_view):
    """backward(a g1 + g2) = a backward(g1) + backward(g2) through the full
    record-parallel path (forward re-walk, coefficients, record kernels,
    chain), float32 arithmetic: compared with the gradient tolerance."""
    cloud, env, res = config2_view
    rng = np.random.default_rng(3)
    g1 = torch.tensor(rng.normal(0, 1e-6, (800, 800, 3)), device="cuda", dtype=torch.float32)
    g2 = torch.tensor(rng.normal(0, 1e-6, (800, 800, 3)), device="cuda", dtype=torch.float32)
    a1, _ = _grads(cloud, res, g1)
    a2, _ = _grads(cloud, res, g2)
    a12, _ = _grads(cloud, res, 3.0 * g1 + g2)
    for k in LINEAR:
        bad, err = grad_close(a12[k], 3.0 * a1[k] + a2[k], rel=1e-3, floor=1e-4)
        assert bad == 0, (k, err)
    # the norm sum is positively homogeneous instead
    a3, _ = _grads(cloud, res, 3.0 * g1)
    assert grad_close(a3["ss_grad"], 3.0 * a1["ss_grad"], rel=1e-4, floor=1e-6)[0] == 0


def test_zero_upstream_gives_zero_gradients(config2_view):
    cloud, env, res = config2_view
    grads, b = _grads(cloud, res, torch.zeros((800, 800, 3), device="cuda", dtype=torch.float32))
    for k in KEYS:
        assert float(grads[k].abs().max()) == 0.0, k
    assert float(b.env_base_log.abs().max()) == 0.0
    # coverage counts do not depend on the upstream gradient
    _, b1 = _grads(cloud, res, torch.ones((800, 800, 3), device="cuda", dtype=torch.float32))
    assert torch.equal(b.touch_count, b1.touch_count)
