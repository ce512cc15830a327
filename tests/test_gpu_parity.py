"""CUDA path vs oracle / reference golden fixtures (needs a B200).

Every call goes through the package API, i.e. through the C ABI of
libss_b200.so.  Tolerances: tile lists, sort orders, cull codes, rects,
nlayers and touched counts bit-exact; images 1e-4 relative (+1e-6 abs);
gradients 1e-3 relative with an array-scaled floor (tests/parity.py).
"""

import numpy as np
import pytest
import torch

from golden_io import SCENES, camera_of, cloud_of, load, proj_of
from parity import grad_close, host, image_close

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _render(d, **over):
    cloud = ss.SurfelCloud.from_host(cloud_of(d))
    cam = ss.Camera(**vars(camera_of(d)))
    env = None
    colors = None
    src = str(d["color_source"])
    if src == "explicit":
        colors = d["colors_in"]
    if "env_base_log" in d:
        env = ss.EnvironmentLight(d["env_base_log"], levels=int(d["env_levels"]))
    opt = ss.RenderOptions(background=tuple(float(v) for v in d["background"]),
                           mip_enabled=bool(d["mip_enabled"]), k_max=int(d["k_max"]), **over)
    return cloud, cam, env, ss.render(cloud, cam, opt, env=env, colors=colors)


@pytest.mark.parametrize("name", SCENES)
def test_preprocess_matches_oracle_bit_exact(name):
    d = load(name)
    cloud, cam, env, res = _render(d)
    ref = O.preprocess(cloud_of(d), camera_of(d), mip_enabled=bool(d["mip_enabled"]))
    got = res.proj
    np.testing.assert_array_equal(host(got.cull_code), ref["cull_code"])
    np.testing.assert_array_equal(host(got.source_index), ref["source_index"])
    np.testing.assert_array_equal(host(got.rect), ref["rect"])
    for k in ("t1", "t2", "t4", "view_z", "eps_z", "sinv", "n_f", "c_cam", "tu_cam", "tv_cam", "jac"):
        np.testing.assert_array_equal(host(getattr(got, k)), ref[k], err_msg=k)
    np.testing.assert_array_equal(host(got.jac_ok), ref["jac_ok"])


@pytest.mark.parametrize("name", SCENES)
def test_tile_lists_bit_exact(name):
    """Tile offsets and sort order equal np.lexsort's on the same records, and
    the reference's own lists whenever the records' rects agree."""
    d = load(name)
    _, _, _, res = _render(d)
    proj = res.proj
    to, pr = O.bin_and_sort(host(proj.rect), host(proj.z_start), proj.width, proj.height)
    np.testing.assert_array_equal(host(res.tile_offsets), to)
    np.testing.assert_array_equal(host(res.pair_rec), pr)
    if np.array_equal(host(proj.rect), d["proj_rect"]):
        np.testing.assert_array_equal(host(res.tile_offsets), d["tile_offsets"])
        np.testing.assert_array_equal(host(res.pair_rec), d["pair_rec"])


@pytest.mark.parametrize("name", SCENES)
def test_forward_images_match_reference(name):
    d = load(name)
    _, _, _, res = _render(d)
    for k in ("rgb", "alpha", "depth"):
        bad, err = image_close(getattr(res, k), d[k])
        assert bad == 0, f"{k}: {bad} pixels off, max abs err {err}"
    np.testing.assert_array_equal(host(res.nlayers), d["nlayers"])
    assert res.stats["discarded_overflow"] == int(d["discarded"])


def test_stacks_and_cover_counts():
    d = load("explicit_cons")
    _, _, _, res = _render(d, collect_stacks=True, with_cover_counts=True)
    np.testing.assert_array_equal(host(res.cover_counts), d["cover_counts"])
    np.testing.assert_array_equal(host(res.stacks["member_count"]), d["stack_member_count"])
    for k in ("weight_sum", "color_sum"):
        bad, err = image_close(res.stacks[k], d[f"stack_{k}"], rel=1e-4, abs_=1e-6)
        assert bad == 0, (k, err)


@pytest.mark.parametrize("path", ["records", "walk"])
@pytest.mark.parametrize("name", SCENES)
def test_backward_matches_reference(name, path):
    d = load(name)
    cloud, cam, env, res = _render(d)
    back = ss.backward_image(cloud, res, g_rgb=d["g_rgb_in"], g_alpha=d.get("g_alpha_in"),
                             cons_scale=float(d["cons_scale"]), path=path)
    for k in ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw", "colors",
              "ss_grad", "env_base_log"):
        if f"g_{k}" not in d:
            continue
        bad, err = grad_close(getattr(back, k), d[f"g_{k}"])
        assert bad == 0, f"{k}: {bad} entries off, max err/scale {err}"
    np.testing.assert_array_equal(host(back.touched), d["g_touched"])
    bad, _ = grad_close(back.background, d["g_background"], rel=1e-4)
    assert bad == 0
    assert back.cons_loss == pytest.approx(float(d["g_cons_loss"]), rel=1e-4, abs=1e-12)


def test_env_refresh_and_adjoint_match_reference():
    d = load("env_ops")
    env = ss.EnvironmentLight(d["base_log"], levels=int(d["levels"]))
    for k in ("base", "diffuse", "specular"):
        bad, err = image_close(getattr(env, k), d[k], rel=1e-5)
        assert bad == 0, (k, err)
    db, dl = env.env_gradient(d["d_diffuse"], d["d_specular"])
    assert grad_close(db, d["d_base"], rel=1e-4)[0] == 0
    assert grad_close(dl, d["d_base_log"], rel=1e-4)[0] == 0
    bad, err = image_close(env.lut, d["lut"], rel=1e-5, abs_=1e-7)
    assert bad == 0, err


def test_env_refresh_from_float64_master():
    """refresh(base_log64=...) (the optimiser's float64 master, like the
    reference's float64 env): the float64 maps follow the reference's own
    float64 computation from the unrounded log radiance."""
    d = load("env_ops")
    env = ss.EnvironmentLight(d["base_log"], levels=int(d["levels"]))
    env.refresh(base_log64=torch.tensor(d["base_log"], device="cuda", dtype=torch.float64))
    for k, k64 in (("base", "base64"), ("diffuse", "diffuse64"), ("specular", "specular64")):
        got, ref = host(getattr(env, k64)), np.asarray(d[k], dtype=np.float64)
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err < 1e-9, (k, err)


def test_empty_and_all_culled():
    cam = ss.Camera.perspective(16, 16, 45.0, (0.0, -3.0, 0.0), (0.0, 0.0, 0.0))
    empty = ss.SurfelCloud(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 2)), np.zeros((0, 3)),
                           np.zeros(0), np.zeros(0))
    opt = ss.RenderOptions(background=(0.4, 0.5, 0.6))
    res = ss.render(empty, cam, opt)
    assert float(res.alpha.abs().max()) == 0.0 and res.stats["pairs"] == 0
    back = ss.backward_image(empty, res, g_rgb=np.ones((16, 16, 3)))
    assert back.centers.shape == (0, 3)
    q = np.array([[1.0, 0.0, 0.0, 0.0]])
    behind = ss.SurfelCloud([[0.0, -10.0, 0.0]], q, np.log([[0.3, 0.3]]), np.zeros((1, 3)), [0.0], [0.0])
    res = ss.render(behind, cam, opt)
    assert int(res.nlayers.max()) == 0
    np.testing.assert_allclose(host(res.rgb), np.broadcast_to(np.float32([0.4, 0.5, 0.6]), (16, 16, 3)))


def test_errors_are_loud():
    d = load("explicit_cons")
    cloud = ss.SurfelCloud.from_host(cloud_of(d))
    cam = ss.Camera(**vars(camera_of(d)))
    bad_colors = d["colors_in"].copy()
    bad_colors[3, 1] = np.nan
    with pytest.raises(ValueError):
        ss.render(cloud, cam, colors=bad_colors)
    with pytest.raises(ValueError):
        ss.render(cloud, cam, ss.RenderOptions(depth_mode="ternary"))
    q = cloud.quats.clone()
    q[0] = 0.0
    zc = ss.SurfelCloud(cloud.centers, q, cloud.log_scales, cloud.albedo_raw, cloud.metallic_raw,
                        cloud.roughness_raw)
    with pytest.raises(ValueError):
        ss.render(zc, cam)


def test_repeat_is_deterministic_forward():
    d = load("config0_small")
    _, _, _, a = _render(d)
    _, _, _, b = _render(d)
    assert torch.equal(a.rgb, b.rgb) and torch.equal(a.pair_rec, b.pair_rec)


def test_fast_coverage_path_is_exact_at_scale():
    """The rasterisers' fast coverage test (FMA + approximate reciprocal with
    an exact fallback near the cut-off) must take the same decision as the
    reference arithmetic for every (pixel, in-rect record) of a config-2 view."""
    import ctypes
    from paper_2605_05876_b200 import _lib, scenes
    from paper_2605_05876_b200.preprocess import run_preprocess
    from paper_2605_05876_b200.rasterizer import bin_state
    cloud = ss.SurfelCloud(**scenes.config2(0, 300_000))
    env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 2))
    lib = _lib.load()
    for cam in ss.fibonacci_cameras(3, 3.5, 800, 800):
        st = run_preprocess(cloud, cam, ss.PreprocessOptions(), _lib.SS_COLOR_IBL, env=env)
        offsets, pair = bin_state(st)
        counts = torch.zeros(3, device="cuda", dtype=torch.int64)
        rc = lib.ss_debug_cover_check(800, 800, 16, _lib.ptr(offsets), _lib.ptr(pair), _lib.ptr(st.pair_rect),
                                      _lib.ptr(st.records), _lib.ptr(counts), _lib.stream_ptr())
        _lib.check(rc, "ss_debug_cover_check")
        n, bad, slow = (int(v) for v in counts.cpu())
        assert n > 1_000_000
        assert bad == 0, f"{bad} coverage decisions differ from the reference arithmetic"
        assert slow < 0.05 * n


def test_tile8_forward_matches_tile16():
    """tile = 8 (two 8x4 warp blocks per tile, a different tile list) renders
    what tile = 16 renders (tile-size invariance, test_rasterizer.py:97-103)."""
    d = load("config0_small")
    _, _, _, res16 = _render(d)
    _, _, _, res8 = _render(d, tile=8)
    bad, err = image_close(res8.rgb, res16.rgb, rel=1e-6, abs_=1e-7)
    assert bad == 0, err
    assert torch.equal(res8.nlayers, res16.nlayers)


@pytest.mark.parametrize("shape", [(8, 16), (12, 24), (9, 15), (64, 128)])
def test_diffuse_quadrature_spectral_and_nbody(shape):
    """The diffuse quadrature (spectral form for even widths, N-body form for
    odd ones) against the dense row-normalised clamped-cosine operator of
    shading.py:275-283 built in float64 here: refresh and its adjoint."""
    he, we = shape
    rng = np.random.default_rng(he * we)
    base_log = rng.normal(0.0, 1.0, (he, we, 3))
    env = ss.EnvironmentLight(base_log, levels=1)
    th = (np.arange(he) + 0.5) * (np.pi / he)
    ph = (np.arange(we) + 0.5) * (2.0 * np.pi / we) - np.pi
    tt, pp = np.meshgrid(th, ph, indexing="ij")
    dirs = np.stack([np.sin(tt) * np.cos(pp), np.sin(tt) * np.sin(pp), np.cos(tt)], -1).reshape(-1, 3)
    solid = (np.sin(tt) * (np.pi / he) * (2.0 * np.pi / we)).reshape(-1)
    D = np.maximum(dirs @ dirs.T, 0.0) * solid[None, :]
    D /= D.sum(axis=1, keepdims=True)
    base = host(env.base64).reshape(-1, 3)
    # device exp vs libm exp: within an ulp or two
    np.testing.assert_allclose(host(env.base64), np.exp(np.asarray(base_log, np.float32).astype(np.float64)),
                               rtol=1e-15, atol=0)
    bad, err = image_close(env.diffuse, (D @ base).reshape(he, we, 3), rel=1e-5, abs_=1e-7)
    assert bad == 0, err
    # the float64 maps the float64 shading reads: the dense product's precision
    # for the spectral form (even widths); the N-body form (odd widths) sums
    # float32 products in float64 chunks
    rtol = 1e-12 if we % 2 == 0 else 1e-6
    np.testing.assert_allclose(host(env.diffuse64), (D @ base).reshape(he, we, 3), rtol=rtol, atol=rtol * 1e-2)
    g = rng.normal(0.0, 1.0, (he, we, 3))
    db, _ = env.env_gradient(g, np.zeros((1, he, we, 3)))
    ref = (D.T @ g.reshape(-1, 3)).reshape(he, we, 3)
    assert grad_close(db, ref, rel=1e-5, floor=1e-6)[0] == 0  # outputs of mixed-sign sums: array-scaled floor
