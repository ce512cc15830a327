"""Pin the CPU oracle (oracle/) against golden fixtures produced by the
reference implementation itself (tests/golden/make_golden.py).

These run without a GPU.  Tolerances:
  * records, tile lists, images, stacks, cover counts: bit-exact when the
    oracle is fed the reference's records (or its numpy float32 scales, the one
    unreproducible SIMD op);
  * float64 gradients: 1e-12 of the array's max magnitude, except quantities
    that pass through numpy's float32 SIMD sigmoid/exp (shading), 1e-6.
"""

import numpy as np
import pytest

from golden_io import SCENES, camera_of, cloud_of, load, proj_of
from oracle import oracle as O

PROJ_FIELDS = ("t1", "t2", "t4", "view_z", "eps_z", "sinv", "n_f", "center_ndc", "jac", "jac_ok",
               "rect", "source_index", "c_cam", "tu_cam", "tv_cam", "cull_code")


def _rel_to_max(a, b):
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", SCENES)
def test_preprocess_bit_exact_given_numpy_scales(name):
    d = load(name)
    cloud, cam = cloud_of(d), camera_of(d)
    got = O.preprocess(cloud, cam, mip_enabled=bool(d["mip_enabled"]),
                       scales=np.exp(cloud.log_scales))
    ref = proj_of(d)
    for k in PROJ_FIELDS:
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)


@pytest.mark.parametrize("name", SCENES)
def test_preprocess_with_own_exp_matches_within_ulps(name):
    d = load(name)
    cloud, cam = cloud_of(d), camera_of(d)
    got = O.preprocess(cloud, cam, mip_enabled=bool(d["mip_enabled"]))
    ref = proj_of(d)
    np.testing.assert_array_equal(got["cull_code"], ref["cull_code"])
    np.testing.assert_array_equal(got["rect"], ref["rect"])
    for k in ("t1", "t2", "t4", "view_z", "eps_z", "c_cam", "tu_cam", "tv_cam"):
        np.testing.assert_allclose(got[k], ref[k], rtol=2e-6, atol=1e-7, err_msg=k)


@pytest.mark.parametrize("name", SCENES)
def test_bin_and_sort_bit_exact(name):
    d = load(name)
    ref = proj_of(d)
    to, pr = O.bin_and_sort(ref["rect"], ref["z_start"], ref["width"], ref["height"])
    np.testing.assert_array_equal(to, d["tile_offsets"])
    np.testing.assert_array_equal(pr, d["pair_rec"])


@pytest.mark.parametrize("name", SCENES)
def test_forward_bit_exact_on_reference_records(name):
    d = load(name)
    cloud, cam = cloud_of(d), camera_of(d)
    res = O.render(cloud, cam, background=d["background"], colors=d["colors"], proj=proj_of(d),
                   k_max=int(d["k_max"]), collect_stacks="stack_weight_sum" in d,
                   with_cover_counts="cover_counts" in d)
    for k in ("rgb", "alpha", "depth", "nlayers"):
        np.testing.assert_array_equal(getattr(res, k), d[k], err_msg=k)
    assert res.discarded == int(d["discarded"])
    if "cover_counts" in d:
        np.testing.assert_array_equal(res.cover_counts, d["cover_counts"])
    if res.stacks is not None:
        for k, v in res.stacks.items():
            np.testing.assert_array_equal(v, d[f"stack_{k}"], err_msg=k)


@pytest.mark.parametrize("name", SCENES)
def test_backward_matches_reference(name):
    d = load(name)
    cloud, cam = cloud_of(d), camera_of(d)
    res = O.render(cloud, cam, background=d["background"], colors=d["colors"], proj=proj_of(d),
                   k_max=int(d["k_max"]))
    env = None
    if "env_base_log" in d:
        env = O.EnvOracle(d["env_base_log"], levels=int(d["env_levels"]))
        np.testing.assert_allclose(env.diffuse, d["env_diffuse"], rtol=1e-12)
        np.testing.assert_allclose(env.specular, d["env_specular"], rtol=1e-12)
    res.color_source = str(d["color_source"])
    g = O.backward_image(cloud, res, d["g_rgb_in"], d.get("g_alpha_in"), float(d["cons_scale"]),
                         env=env)
    shaded = res.color_source != "explicit"
    for k in ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw",
              "colors", "ss_grad", "background", "env_base_log"):
        if f"g_{k}" not in d:
            continue
        sim = shaded and k not in ("log_scales", "colors", "ss_grad", "background")
        tol = 1e-6 if sim else 1e-12
        assert _rel_to_max(g[k], d[f"g_{k}"]) <= tol, k
    np.testing.assert_array_equal(g["touched"], d["g_touched"])
    assert g["cons_loss"] == pytest.approx(float(d["g_cons_loss"]), rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("name", ["ibl_env", "config0_small"])
def test_shading_colors_match(name):
    d = load(name)
    cloud, cam = cloud_of(d), camera_of(d)
    env = O.EnvOracle(d["env_base_log"], levels=int(d["env_levels"]))
    cols = O.shade(cloud, env, cam)
    np.testing.assert_allclose(cols, d["colors"], rtol=2e-6, atol=1e-7)


def test_end_to_end_render_config0_small():
    """Full oracle pipeline (own preprocess + own shading) against the
    reference render: tile lists bit-exact, images within 1e-5."""
    d = load("config0_small")
    cloud, cam = cloud_of(d), camera_of(d)
    env = O.EnvOracle(d["env_base_log"], levels=int(d["env_levels"]))
    res = O.render(cloud, cam, env=env)
    np.testing.assert_array_equal(res.tile_offsets, d["tile_offsets"])
    np.testing.assert_array_equal(res.pair_rec, d["pair_rec"])
    np.testing.assert_array_equal(res.nlayers, d["nlayers"])
    np.testing.assert_allclose(res.rgb, d["rgb"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(res.alpha, d["alpha"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(res.depth, d["depth"], rtol=1e-5, atol=1e-6)
    val, g = O.photometric_l1(res.rgb, d["target"])
    assert val == pytest.approx(float(d["loss_value"]), rel=1e-5)


def test_env_operators_and_lut():
    d = load("env_ops")
    env = O.EnvOracle(d["base_log"], levels=int(d["levels"]))
    np.testing.assert_allclose(env.base, d["base"], rtol=1e-15)
    np.testing.assert_allclose(env.diffuse, d["diffuse"], rtol=1e-12)
    np.testing.assert_allclose(env.specular, d["specular"], rtol=1e-12)
    d_base, d_log = env.env_gradient(d["d_diffuse"], d["d_specular"])
    assert _rel_to_max(d_base, d["d_base"]) < 1e-12
    assert _rel_to_max(d_log, d["d_base_log"]) < 1e-12
    lut = O.brdf_lut(64, 128)
    np.testing.assert_allclose(lut, d["lut"], rtol=1e-6, atol=1e-7)


def test_adam_trace():
    d = load("optim_refine")
    p = d["adam_p0"].copy()
    m = np.zeros(p.shape); v = np.zeros(p.shape)
    for k in range(3):
        O.adam_step(p, d["adam_grads"][k], m, v, k + 1, 0.01)
        np.testing.assert_array_equal(p, d["adam_traj"][k])


def test_refine_topology():
    d = load("optim_refine")
    cloud = cloud_of(d)
    keep, split_rows, index_map, reasons = O.refine_topology(
        cloud.centers, cloud.quats, cloud.log_scales, d["grad_sum"], d["view_count"],
        d["mean_dist"], int(d["max_surfels"]), quantile=0.9)
    np.testing.assert_array_equal(index_map, d["index_map"])
    assert [reasons[k] for k in ("stale", "isolated", "floater", "split")] == list(d["reasons"])
    kept_idx = np.flatnonzero(keep)
    parents = kept_idx[split_rows]
    cp, cm, cls = O.split_children(cloud.centers, cloud.quats, cloud.log_scales, parents)
    ns = len(split_rows)
    n_new = len(d["new_centers"])
    # children offsets use exp(log_scales) (numpy float32 SIMD exp): ulp-level
    np.testing.assert_allclose(cp, d["new_centers"][n_new - 2 * ns:n_new - ns], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(cm, d["new_centers"][n_new - ns:], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(cls, d["new_log_scales"][n_new - ns:], rtol=1e-6)


def test_loss_oracle_matches_reference_goldens():
    """oracle tone_map / ssim_loss / photometric_loss / silhouette_loss vs the
    reference's own outputs (tests/golden/make_golden_losses.py)."""
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "losses.npz"))
    x, y, g_up = d["img"], d["tgt"], d["g_up"]
    for mode in ("ldr", "hdr-loss"):
        k = mode.replace("-", "_")
        np.testing.assert_allclose(O.tone_map(x, mode), d["tone_" + k], rtol=1e-15, atol=0)
        np.testing.assert_allclose(O.tone_map_backward(x, mode, g_up), d["tone_bwd_" + k], rtol=1e-15, atol=0)
        for lam in (0.0, 0.2):
            v, g = O.photometric_loss(O.tone_map(x, mode), O.tone_map(y, mode), lam)
            assert v == pytest.approx(float(d[f"photo_{k}_{int(lam * 10)}"]), rel=1e-14)
            np.testing.assert_allclose(g, d[f"photo_grad_{k}_{int(lam * 10)}"], rtol=1e-10, atol=1e-17)
    v, g = O.ssim_loss(x, y)
    assert v == pytest.approx(float(d["ssim"]), rel=1e-14)
    np.testing.assert_allclose(g, d["ssim_grad"], rtol=1e-10, atol=1e-16)
    v, g = O.ssim_loss(d["alpha"], d["mask"])
    assert v == pytest.approx(float(d["ssim_1c"]), rel=1e-14)
    np.testing.assert_allclose(g, d["ssim_1c_grad"], rtol=1e-10, atol=1e-16)
    v, g = O.silhouette_loss(d["alpha"], d["mask"])
    assert v == pytest.approx(float(d["sil"]), rel=1e-14)
    np.testing.assert_allclose(g, d["sil_grad"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("name", ["sphere", "shell"])
def test_knn_oracle_matches_reference_goldens(name):
    """oracle knn_oriented / normal_consistency vs the reference NeighborIndex
    (scipy cKDTree) and normal_consistency_loss (tests/golden/make_golden_knn.py)."""
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "knn.npz"))
    nb, md = O.knn_oriented(d[f"{name}_centers"], d[f"{name}_quats"], k=8)
    np.testing.assert_array_equal(nb, d[f"{name}_neighbors"])
    np.testing.assert_allclose(md, d[f"{name}_mean_dist"], rtol=1e-14, atol=0)
    loss, g = O.normal_consistency(d[f"{name}_centers"], d[f"{name}_quats"], nb, md)
    assert loss == pytest.approx(float(d[f"{name}_nc_loss"]), rel=1e-13)
    np.testing.assert_allclose(g, d[f"{name}_nc_grad"], rtol=1e-9, atol=1e-16)


def test_refine_oracle_tree_path_matches_brute_force():
    """The oracle's refine_topology switches to the reference's own cKDTree
    isolation query above 4000 surfels (densify.py:119-121); both paths give
    the same plan on the same input."""
    rng = np.random.default_rng(3)
    n = 3000
    c = rng.normal(size=(n, 3)).astype(np.float32)
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    c[:20] *= 3.0
    q = rng.normal(size=(n, 4)).astype(np.float32)
    ls = np.log(rng.uniform(0.01, 0.05, (n, 2))).astype(np.float32)
    gs = rng.exponential(1e-4, n)
    gs[rng.uniform(size=n) < 0.1] = 0.0
    vc = rng.integers(0, 5, n)
    mnd = rng.uniform(0.01, 0.04, n)
    a = O.refine_topology(c, q, ls, gs, vc, mnd, int(1.02 * n), quantile=0.95)
    big = np.concatenate([c, c + 100.0])  # a far copy: > 4000 rows takes the tree path
    b = O.refine_topology(big, np.concatenate([q, q]), np.concatenate([ls, ls]), np.concatenate([gs, gs]),
                          np.concatenate([vc, vc]), np.concatenate([mnd, mnd]), int(2.04 * n), quantile=0.95)
    assert np.array_equal(b[0][:n], a[0]) and b[3]["isolated"] == 2 * a[3]["isolated"]
