"""Boundary behaviour of the drop-in API (needs a B200): proj= reuse,
bin_and_sort on a ProjectedSurfels, the pair-capacity clamp, the float64
optimiser state, the caller-owned env operators."""

import numpy as np
import pytest
import torch

from golden_io import SCENES, camera_of, cloud_of, load
from parity import grad_close, host

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_05876_b200 import _lib, scenes, shading  # noqa: E402
from paper_2605_05876_b200.preprocess import run_preprocess  # noqa: E402


def _scene(name):
    d = load(name)
    cloud = ss.SurfelCloud.from_host(cloud_of(d))
    cam = ss.Camera(**vars(camera_of(d)))
    env = ss.EnvironmentLight(d["env_base_log"], levels=int(d["env_levels"])) if "env_base_log" in d else None
    colors = d["colors_in"] if str(d["color_source"]) == "explicit" else None
    opt = ss.RenderOptions(background=tuple(float(v) for v in d["background"]),
                           mip_enabled=bool(d["mip_enabled"]), k_max=int(d["k_max"]))
    return d, cloud, cam, env, colors, opt


@pytest.mark.parametrize("name", SCENES)
def test_bin_and_sort_on_projected_surfels(name):
    """bin_and_sort(preprocess(...)) -- the reference's own call sequence
    (rasterizer.py:92-116) -- gives np.lexsort's tile lists bit for bit."""
    d, cloud, cam, env, colors, opt = _scene(name)
    proj = ss.preprocess(cloud, cam, opt.preprocess_options())
    offsets, pair_rec, ntx, nty = ss.bin_and_sort(proj)
    to, pr = O.bin_and_sort(host(proj.rect), host(proj.z_start), proj.width, proj.height)
    np.testing.assert_array_equal(host(offsets), to)
    np.testing.assert_array_equal(host(pair_rec), pr)
    assert ntx * nty == len(to) - 1
    if np.array_equal(host(proj.rect), d["proj_rect"]):
        np.testing.assert_array_equal(host(pair_rec), d["pair_rec"])


@pytest.mark.parametrize("name", SCENES)
def test_render_with_proj_reuse(name):
    """render(..., proj=preprocess(...)) rasterises the given projection:
    identical to a render that projects itself, and so is its backward."""
    d, cloud, cam, env, colors, opt = _scene(name)
    a = ss.render(cloud, cam, opt, env=env, colors=colors)
    proj = ss.preprocess(cloud, cam, opt.preprocess_options())
    b = ss.render(cloud, cam, opt, env=env, colors=colors, proj=proj)
    assert b.proj is proj
    for k in ("rgb", "alpha", "depth", "nlayers", "pair_rec", "tile_offsets"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    g = torch.tensor(np.random.default_rng(3).normal(size=tuple(a.rgb.shape)), device="cuda", dtype=torch.float32)
    ga, gb = ss.backward_image(cloud, a, g_rgb=g), ss.backward_image(cloud, b, g_rgb=g)
    for k in ("centers", "quats", "log_scales", "albedo_raw"):
        assert grad_close(getattr(gb, k), getattr(ga, k), rel=1e-6, floor=1e-9)[0] == 0, k


def test_render_proj_size_mismatch_raises():
    d, cloud, cam, env, colors, opt = _scene("albedo_nomip")
    proj = ss.preprocess(cloud, cam, opt.preprocess_options())
    small = ss.Camera(**{**vars(camera_of(d)), "width": int(cam.width) // 2})
    with pytest.raises(ValueError):
        ss.render(cloud, small, opt, proj=proj)


def test_pair_capacity_overflow_is_clamped_and_flagged():
    """With pair buffers smaller than the view needs, the binning flags the
    overflow, reports the pairs needed, and clamps the tile offsets to the
    capacity so the rasteriser never reads past the buffers."""
    gt = scenes.config0(0, 3000)
    cloud = ss.SurfelCloud(**gt)
    cam = ss.Camera.perspective(96, 96, 40.0, (3.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    st = run_preprocess(cloud, cam, ss.PreprocessOptions(), _lib.SS_COLOR_ALBEDO)
    need = int(st.tile_counts.sum().item())
    cap = need // 3
    lib = _lib.load()
    dev = st.records.device
    offsets = torch.empty(st.ntiles + 1, device=dev, dtype=torch.int32)
    cursors = torch.empty(st.ntiles, device=dev, dtype=torch.int32)
    keys = torch.empty(cap, device=dev, dtype=torch.int64)
    pair = torch.full((cap,), -1, device=dev, dtype=torch.int32)
    rects = torch.empty((cap, 2), device=dev, dtype=torch.int32)
    _lib.check(lib.ss_bin_sort(len(cloud), _lib.ptr(st.bininfo), _lib.ptr(st.cull), 96, 96, 16,
                               _lib.ptr(st.tile_counts), _lib.ptr(offsets), _lib.ptr(cursors), _lib.ptr(keys),
                               _lib.ptr(pair), _lib.ptr(rects), cap, _lib.ptr(st.flags), None, _lib.stream_ptr()),
               "ss_bin_sort")
    flags = host(st.flags)
    off = host(offsets)
    assert flags[2] == 1 and flags[3] == need
    assert off.max() <= cap and off[-1] == cap and (np.diff(off) >= 0).all()
    pr = host(pair)
    assert ((pr >= 0) & (pr < len(cloud))).all()
    # the forward over the clamped lists stays in bounds
    rgb = torch.empty((96, 96, 3), device=dev)
    a = torch.empty((96, 96), device=dev)
    z = torch.empty((96, 96), device=dev)
    nl = torch.empty((96, 96), device=dev, dtype=torch.int32)
    bg, _k = _lib.fvec((0.0, 0.0, 0.0))
    _lib.check(lib.ss_raster_forward(96, 96, 16, _lib.ptr(offsets), _lib.ptr(pair), _lib.ptr(rects),
                                     _lib.ptr(st.records), bg, 16, _lib.ptr(rgb), _lib.ptr(a), _lib.ptr(z), _lib.ptr(nl),
                                     None, None, None, _lib.stream_ptr()), "ss_raster_forward")
    torch.cuda.synchronize()
    assert torch.isfinite(rgb).all()


def test_env_operators_are_caller_owned():
    """The library holds no env state: two shapes refreshed alternately give
    the same maps as refreshing each alone (no process-global operator)."""
    a = ss.EnvironmentLight(np.log(scenes.env_lognormal(16, 32, 1)))
    b = ss.EnvironmentLight(np.log(scenes.env_lognormal(32, 64, 2)))
    sa, sb = a.specular.clone(), b.specular.clone()
    da, db = a.diffuse.clone(), b.diffuse.clone()
    for _ in range(2):
        a.refresh()
        b.refresh()
    assert torch.equal(a.specular, sa) and torch.equal(b.specular, sb)
    assert torch.equal(a.diffuse, da) and torch.equal(b.diffuse, db)
    ops = shading.env_ops(16, 32)
    assert ops.khat is not None and ops.khat.numel() == _lib.load().ss_env_khat_words(16, 32)
