"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \
        SURFSPLAT_CACHE_DIR=/tmp/ssc python tests/golden/make_golden.py

Every fixture stores the seeded inputs together with the reference's own
outputs (surfsplat 0.1.0: preprocess / bin_and_sort / render / backward_image /
EnvironmentLight / brdf_lut / Adam / refine_topology).  The committed .npz
files pin ``oracle/`` (tests/test_oracle_golden.py) which in turn is the
checker for the CUDA path.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_cache")
os.environ.setdefault("SURFSPLAT_CACHE_DIR", "/tmp/ss_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from surfsplat.adam import Adam  # noqa: E402
from surfsplat.backward import backward_image  # noqa: E402
from surfsplat.camera import Camera  # noqa: E402
from surfsplat.densify import DensifyStats, refine_topology  # noqa: E402
from surfsplat.losses import photometric_loss  # noqa: E402
from surfsplat.rasterizer import RenderOptions, render  # noqa: E402
from surfsplat.shading import EnvironmentLight, brdf_lut  # noqa: E402
from surfsplat.surfels import SurfelCloud, logit, quats_from_normals  # noqa: E402

CLOUD_KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw")
PROJ_KEYS = ("t1", "t2", "t4", "view_z", "eps_z", "sinv", "n_f", "center_ndc", "jac", "jac_ok",
             "rect", "source_index", "c_cam", "tu_cam", "tv_cam", "cull_code")
GRAD_KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw",
             "colors", "background", "ss_grad", "touched")


def random_cloud(n, seed, box=0.8, scale_range=(0.08, 0.3)):
    rng = np.random.default_rng(seed)
    return SurfelCloud(
        centers=rng.uniform(-box, box, size=(n, 3)).astype(np.float32),
        quats=rng.normal(size=(n, 4)).astype(np.float32),
        log_scales=np.log(rng.uniform(*scale_range, size=(n, 2))).astype(np.float32),
        albedo_raw=rng.normal(0.0, 1.0, size=(n, 3)).astype(np.float32),
        metallic_raw=rng.normal(0.0, 1.0, size=n).astype(np.float32),
        roughness_raw=rng.normal(0.0, 1.0, size=n).astype(np.float32),
    )


def random_camera(seed, width, height, radius=3.2, fov=45.0):
    rng = np.random.default_rng(seed)
    az = rng.uniform(0.0, 2.0 * np.pi)
    el = rng.uniform(-0.9, 0.9)
    eye = radius * np.array([np.cos(az) * np.cos(el), np.sin(az) * np.cos(el), np.sin(el)])
    return Camera.perspective(width, height, fov, eye, (0.0, 0.0, 0.0))


def config0_cloud(n, seed):
    """BASELINE config 0 geometry: unit sphere, radial normals."""
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(n, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    ls = rng.uniform(np.log(0.01), np.log(0.03), size=(n, 2))
    alb = rng.uniform(0, 1, size=(n, 3))
    rough = rng.uniform(0.1, 0.9, size=n)
    met = rng.uniform(0, 1, size=n)
    cl = lambda x: logit(np.clip(x, 1e-5, 1 - 1e-5))
    return SurfelCloud(centers=p.astype(np.float32), quats=quats_from_normals(p).astype(np.float32),
                       log_scales=ls.astype(np.float32), albedo_raw=cl(alb).astype(np.float32),
                       metallic_raw=cl(met).astype(np.float32), roughness_raw=cl(rough).astype(np.float32))


def pack_cloud(prefix, cloud):
    return {f"{prefix}{k}": np.asarray(getattr(cloud, k)) for k in CLOUD_KEYS}


def pack_camera(cam):
    return {"cam_view": cam.view, "cam_proj": cam.proj, "cam_wh": np.array([cam.width, cam.height])}


def pack_render(res):
    out = {f"proj_{k}": np.asarray(getattr(res.proj, k)) for k in PROJ_KEYS}
    out.update({"rgb": res.rgb, "alpha": res.alpha, "depth": res.depth, "nlayers": res.nlayers,
                "colors": res.colors, "tile_offsets": res.tile_offsets, "pair_rec": res.pair_rec,
                "discarded": np.int64(res.stats["discarded_overflow"])})
    if res.cover_counts is not None:
        out["cover_counts"] = res.cover_counts
    if res.stacks is not None:
        for k, v in res.stacks.items():
            out[f"stack_{k}"] = v
    return out


def pack_grads(back):
    out = {f"g_{k}": np.asarray(getattr(back, k)) for k in GRAD_KEYS}
    out["g_cons_loss"] = np.float64(back.cons_loss)
    if back.env_base_log is not None:
        out["g_env_base_log"] = back.env_base_log
    return out


def scene_fixture(name, cloud, cam, opt, env=None, colors=None, cons_scale=0.0, seed=0,
                  loss="random"):
    res = render(cloud, cam, opt, env=env, colors=colors)
    rng = np.random.default_rng(seed)
    if loss == "random":
        g_rgb = rng.normal(size=res.rgb.shape)
        g_alpha = rng.normal(size=res.alpha.shape)
        extra = {}
    else:  # config-0 L1 against a perturbed-position target
        tcloud = cloud.copy()
        tcloud.centers = (cloud.centers + rng.normal(0, 0.01, cloud.centers.shape)).astype(np.float32)
        target = render(tcloud, cam, opt, env=env, colors=colors).rgb
        val, g_rgb = photometric_loss(res.rgb, target, lambda_ssim=0.0)
        g_alpha = None
        extra = {"target": target, "loss_value": np.float64(val), "target_centers": tcloud.centers}
    back = backward_image(cloud, res, g_rgb=g_rgb, g_alpha=g_alpha, cons_scale=cons_scale)
    data = {**pack_cloud("cloud_", cloud), **pack_camera(cam), **pack_render(res), **pack_grads(back),
            **extra, "g_rgb_in": g_rgb, "cons_scale": np.float64(cons_scale),
            "background": np.asarray(opt.background, np.float32),
            "mip_enabled": np.int64(opt.mip_enabled), "color_source": np.array(res.color_source),
            "k_max": np.int64(opt.k_max)}
    if g_alpha is not None:
        data["g_alpha_in"] = g_alpha
    if colors is not None:
        data["colors_in"] = np.asarray(colors, np.float32)
    if env is not None:
        data["env_base_log"] = env.base_log
        data["env_levels"] = np.int64(env.levels)
        data["env_diffuse"] = env.diffuse
        data["env_specular"] = env.specular
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **data)
    print(f"{name}: N={len(cloud)} P={len(res.pair_rec)} -> {os.path.getsize(path)} B")


def main():
    # 1. explicit colours, consolidation on, MIP on
    cloud = random_cloud(40, 100)
    cam = random_camera(101, 40, 36)
    colors = np.random.default_rng(102).uniform(0, 1, (40, 3))
    scene_fixture("explicit_cons", cloud, cam,
                  RenderOptions(background=(0.15, 0.05, 0.25), collect_stacks=True,
                                with_cover_counts=True),
                  colors=colors, cons_scale=0.5 / (40 * 36), seed=103)
    # 2. MIP off, albedo colour source
    cloud = random_cloud(60, 200)
    cam = random_camera(201, 48, 40)
    scene_fixture("albedo_nomip", cloud, cam, RenderOptions(mip_enabled=False), seed=203)
    # 3. IBL shading with a small env (full shading + env adjoint)
    cloud = random_cloud(50, 300)
    cam = random_camera(301, 40, 40)
    env = EnvironmentLight(base_log=np.random.default_rng(302).normal(np.log(0.6), 0.3, (8, 16, 3)))
    scene_fixture("ibl_env", cloud, cam, RenderOptions(background=(0.1, 0.2, 0.3)), env=env,
                  cons_scale=0.25 / 1600, seed=303)
    # 4. K_MAX stop: 24 stacked parallel surfels (test_rasterizer.py:216-231)
    n = 24
    centers = np.zeros((n, 3))
    centers[:, 1] = np.arange(n) * 0.8
    normals = np.tile([0.0, -1.0, 0.0], (n, 1))
    cloud = SurfelCloud.from_oriented_points(centers, normals, 0.5)
    cam = Camera.perspective(33, 33, 45.0, (0.0, -5.0, 0.0), (0.0, 0.0, 0.0))
    colors = np.random.default_rng(5).uniform(0, 1, (n, 3))
    scene_fixture("kmax_stack", cloud, cam, RenderOptions(collect_stacks=True), colors=colors,
                  cons_scale=1.0 / (33 * 33), seed=403)
    # 5. culling: behind, offscreen, non-finite, near plane, plus normal rows
    cloud = random_cloud(32, 500)
    cam = random_camera(501, 32, 32)
    pos = cam.position
    c = cloud.centers.copy()
    c[0] = (pos * 2.0).astype(np.float32)            # behind the camera
    c[1] = (pos * 0.9999).astype(np.float32)          # at the eye: near plane / behind
    c[2] = np.array([30.0, 30.0, 30.0], np.float32)   # far off-axis
    c[3, 0] = np.nan                                   # non-finite
    ls = cloud.log_scales.copy()
    ls[4] = np.log(2.5)                                # huge surfel close to the camera
    c[4] = (pos * 0.85).astype(np.float32)
    cloud.centers = c
    cloud.log_scales = ls
    colors = np.random.default_rng(502).uniform(0, 1, (32, 3))
    scene_fixture("culling", cloud, cam, RenderOptions(), colors=colors, seed=503)
    # 6. config-0 workload at reduced size: 2000 surfels on the unit sphere, 64^2, 16x32 env, L1
    cloud = config0_cloud(2000, 600)
    cam = Camera.perspective(64, 64, 40.0, (3.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    rng = np.random.default_rng(601)
    env = EnvironmentLight.from_base(np.exp(rng.normal(0.0, 1.0, (16, 32, 3))))
    scene_fixture("config0_small", cloud, cam, RenderOptions(), env=env, seed=602, loss="l1")

    # 7. environment operators and the BRDF LUT
    rng = np.random.default_rng(700)
    env = EnvironmentLight(base_log=rng.normal(0.0, 0.5, (8, 16, 3)))
    d_diff = rng.normal(size=(8, 16, 3))
    d_spec = rng.normal(size=(env.levels, 8, 16, 3))
    d_base, d_log = env.env_gradient(d_diff, d_spec)
    np.savez_compressed(os.path.join(HERE, "env_ops.npz"), base_log=env.base_log, levels=env.levels,
                        base=env.base, diffuse=env.diffuse, specular=env.specular,
                        d_diffuse=d_diff, d_specular=d_spec, d_base=d_base, d_base_log=d_log,
                        lut=brdf_lut(64, 128, cache_dir="/tmp/ss_lut_golden"))
    print("env_ops")

    # 8. Adam trace (adam.py) and one refinement pass (densify.py)
    rng = np.random.default_rng(800)
    p0 = rng.normal(size=(17, 3)).astype(np.float32)
    grads = rng.normal(size=(3, 17, 3))
    opt = Adam()
    p = p0.copy()
    traj = []
    for k in range(3):
        opt.step("x", p, grads[k], 0.01)
        traj.append(p.copy())
    cloud = random_cloud(200, 801, box=0.5, scale_range=(0.01, 0.06))
    gs = np.abs(rng.normal(size=200)) * (rng.uniform(size=200) > 0.1)
    vc = rng.integers(0, 5, size=200)
    mean_dist = rng.uniform(0.005, 0.05, size=200)
    stats = DensifyStats(gs.astype(np.float64), vc.astype(np.int64))
    new_cloud, index_map, reasons = refine_topology(cloud, stats, mean_dist, max_surfels=230,
                                                    quantile=0.9)
    np.savez_compressed(os.path.join(HERE, "optim_refine.npz"), adam_p0=p0, adam_grads=grads,
                        adam_traj=np.stack(traj), **pack_cloud("cloud_", cloud), grad_sum=gs,
                        view_count=vc, mean_dist=mean_dist, max_surfels=230,
                        **pack_cloud("new_", new_cloud), index_map=index_map,
                        reasons=np.array([reasons["stale"], reasons["isolated"],
                                          reasons["floater"], reasons["split"]]))
    print("optim_refine", reasons)


if __name__ == "__main__":
    main()
