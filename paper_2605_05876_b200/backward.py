"""backward_image() API (mirror of surfsplat.backward, backward.py:29-470).

Without the consolidation term (cons_scale = 0, the common case) the image
gradient goes through the training step's walk-free kernels: deferred-loss
forward (layer sums + closing depths), ss_train_coefs (suffix recursion with
g_rgb and g_alpha) and the record-parallel backward.  With cons_scale > 0 the
replaying tile-CTA backward (pixel replays, per-layer suffix recursion,
consolidation, warp-reduced per-record atomics) runs instead.  Then the
per-surfel chain kernel (MIP chain, rows -> world, shading adjoint with the
derived-map scatter, quaternion adjoint); with IBL colours the env adjoint
kernel finishes the environment gradient.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .preprocess import make_opts


@dataclass
class BackwardResult:
    centers: torch.Tensor
    quats: torch.Tensor
    log_scales: torch.Tensor
    albedo_raw: torch.Tensor
    metallic_raw: torch.Tensor
    roughness_raw: torch.Tensor
    colors: torch.Tensor
    env_base_log: torch.Tensor | None
    background: torch.Tensor
    ss_grad: torch.Tensor
    touched: torch.Tensor
    cons_loss: float
    touch_count: torch.Tensor | None = None
    d_diffuse: torch.Tensor | None = None
    d_specular: torch.Tensor | None = None


def zero_grads(n, dev):
    z = lambda *s: torch.zeros(s, device=dev, dtype=torch.float32)
    return {"centers": z(n, 3), "quats": z(n, 4), "log_scales": z(n, 2), "albedo_raw": z(n, 3),
            "metallic_raw": z(n), "roughness_raw": z(n), "colors": z(n, 3), "ss_grad": z(n),
            "touched": torch.zeros(n, device=dev, dtype=torch.int32)}


def grads_struct(g, d_diffuse=None, d_specular=None, d_diffuse4=None, d_specular4=None):
    return _lib.SsGrads(*(_lib.ptr(g[k]) for k in ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw",
                                                   "roughness_raw")),
                        _lib.ptr(g.get("colors")), _lib.ptr(g["ss_grad"]), _lib.ptr(g["touched"]),
                        _lib.ptr(d_diffuse), _lib.ptr(d_specular), _lib.ptr(d_diffuse4), _lib.ptr(d_specular4))


def _record_backward(lib, result, g_rgb, g_alpha, acc, acc64, bgp, cons_scale=0.0, cons=None):
    """The walk-free backward of the training step for an API render: the
    deferred-loss forward re-derives the per-pixel layer sums and closing
    depths, ss_train_coefs turns them into the layer coefficients for (g_rgb,
    g_alpha), and the record-parallel kernel fills the per-record accumulator
    (DESIGN.md §4).  With cons_scale > 0 the forward also parks the layer
    depth moments, ss_train_coefs_cons adds the consolidation penalty
    (value into `cons`) and the record kernels its depth / weight terms."""
    st, opt, cam = result.state, result.options, result.camera
    dev = st.records.device
    H, W, K = int(cam.height), int(cam.width), int(opt.k_max)
    f32 = dict(device=dev, dtype=torch.float32)
    coef = torch.empty(9 * K * H * W, **f32)  # float4 planes, A_lo planes, raw-sum lo planes
    thr = torch.empty((K, H * W), **f32)
    hdr = torch.empty((H * W, 8), device=dev, dtype=torch.int32)
    rgb = torch.empty((H, W, 3), **f32)
    n = st.records.shape[0]
    scratch = torch.empty(lib.ss_train_backward_scratch_words(n, W, H), **f32)
    if float(cons_scale) > 0.0:
        zst = torch.empty((K, H * W, 4), **f32)
        _lib.check(lib.ss_train_forward_zstats(W, H, int(opt.tile), _lib.ptr(result.tile_offsets32),
                                               _lib.ptr(result.pair_src), _lib.ptr(st.pair_rect), _lib.ptr(st.records),
                                               bgp, K, _lib.ptr(coef), _lib.ptr(thr), _lib.ptr(hdr), _lib.ptr(rgb), None,
                                               None, _lib.ptr(zst), _lib.stream_ptr()), "ss_train_forward_zstats")
        _lib.check(lib.ss_train_coefs_cons(W, H, K, _lib.ptr(hdr), _lib.ptr(coef), _lib.ptr(zst), _lib.ptr(g_rgb),
                                           None, _lib.ptr(g_alpha), bgp, float(cons_scale), _lib.ptr(cons),
                                           _lib.stream_ptr()), "ss_train_coefs_cons")
        _lib.check(lib.ss_train_backward_records_cons(n, _lib.ptr(st.cull), _lib.ptr(st.records), W, H, K,
                                                      _lib.ptr(coef), _lib.ptr(thr), _lib.ptr(hdr), _lib.ptr(zst),
                                                      _lib.ptr(scratch), _lib.ptr(acc), _lib.ptr(acc64),
                                                      _lib.stream_ptr()), "ss_train_backward_records_cons")
        return
    _lib.check(lib.ss_train_forward(W, H, int(opt.tile), _lib.ptr(result.tile_offsets32), _lib.ptr(result.pair_src),
                                    _lib.ptr(st.pair_rect), _lib.ptr(st.records), bgp, K, None, _lib.ptr(coef),
                                    _lib.ptr(thr), _lib.ptr(hdr), None, _lib.ptr(rgb), None, None, _lib.stream_ptr()),
               "ss_train_forward")
    _lib.check(lib.ss_train_coefs(W, H, K, _lib.ptr(hdr), _lib.ptr(coef), _lib.ptr(g_rgb), None, _lib.ptr(g_alpha),
                                  bgp, _lib.stream_ptr()), "ss_train_coefs")
    _lib.check(lib.ss_train_backward_records(n, _lib.ptr(st.cull), _lib.ptr(st.records), W, H, K, _lib.ptr(coef),
                                             _lib.ptr(thr), _lib.ptr(hdr), _lib.ptr(scratch), _lib.ptr(acc),
                                             _lib.ptr(acc64), _lib.stream_ptr()), "ss_train_backward_records")


def backward_image(cloud, result, g_rgb=None, g_alpha=None, cons_scale=0.0, path="records") -> BackwardResult:
    """backward.py:324-470.  path: "records" (default) -- the walk-free
    record-parallel kernels of the training step; "walk" -- the replaying
    tile backward (ss_raster_backward, the reference's own two-pass order)."""
    if path not in ("records", "walk"):
        raise ValueError("path must be 'records' or 'walk'")
    opt = result.options
    if opt.depth_mode != "interval":
        raise ValueError("backward requires depth_mode='interval'")
    if result.state is None:
        raise ValueError("result was not produced by paper_2605_05876_b200.render")
    lib = _lib.load()
    st = result.state
    dev = st.records.device
    cam = result.camera
    H, W = int(cam.height), int(cam.width)
    n = len(cloud)
    g_rgb = torch.zeros((H, W, 3), device=dev) if g_rgb is None else torch.as_tensor(g_rgb, device=dev)
    g_rgb = g_rgb.to(torch.float32).contiguous()
    ga = None if g_alpha is None else torch.as_tensor(g_alpha, device=dev).to(torch.float32).contiguous()
    acc = torch.zeros((n, _lib.ACC_FLOATS), device=dev, dtype=torch.float32)
    acc64 = None
    cons = torch.zeros(1, device=dev, dtype=torch.float64)
    bgp, _keep = _lib.fvec(opt.background)
    if not float(cons_scale) >= 0.0:
        raise ValueError("cons_scale must be >= 0")
    if path == "records":
        acc64 = torch.empty((n, _lib.ACC64_WIDTH), device=dev, dtype=torch.float64)
        _record_backward(lib, result, g_rgb, ga, acc, acc64, bgp, cons_scale, cons)
    else:
        rc = lib.ss_raster_backward(W, H, int(opt.tile), _lib.ptr(result.tile_offsets32), _lib.ptr(result.pair_src),
                                    _lib.ptr(st.pair_rect), _lib.ptr(st.records), bgp, int(opt.k_max), _lib.ptr(g_rgb),
                                    _lib.ptr(ga), float(cons_scale), _lib.ptr(acc), _lib.ptr(cons), _lib.stream_ptr())
        _lib.check(rc, "ss_raster_backward")
    g = zero_grads(n, dev)
    env = result.env
    ibl = result.color_source == "ibl"
    d_diff = d_spec = d_diff4 = d_spec4 = None
    if ibl:
        d_diff = torch.zeros(env.base.shape, device=dev, dtype=torch.float64)
        d_spec = torch.zeros(env.specular.shape, device=dev, dtype=torch.float64)
        # float32 accumulators with 16-byte texels for the scatter, folded in below
        d_diff4 = torch.zeros((*env.base.shape[:2], 4), device=dev, dtype=torch.float32)
        d_spec4 = torch.zeros((*env.specular.shape[:3], 4), device=dev, dtype=torch.float32)
    source = {"explicit": _lib.SS_COLOR_EXPLICIT, "ibl": _lib.SS_COLOR_IBL, "albedo": _lib.SS_COLOR_ALBEDO}[result.color_source]
    cl = _lib.make_cloud(cloud)
    camst = _lib.make_camera(cam)
    po = make_opts(opt.preprocess_options(), int(opt.tile))
    envs = _lib.make_env(env) if ibl else None
    gs = grads_struct(g, d_diff, d_spec, d_diff4, d_spec4)
    rc = lib.ss_chain_backward(ctypes.byref(cl), ctypes.byref(camst), ctypes.byref(po), source,
                               ctypes.byref(envs) if envs is not None else None, _lib.ptr(st.cull), _lib.ptr(acc),
                               _lib.ptr(acc64), _lib.ptr(st.aux.get("cells_packed") if ibl else None),
                               ctypes.byref(gs), _lib.stream_ptr())
    _lib.check(rc, "ss_chain_backward")
    g_env = None
    if ibl:
        for src, dst in ((d_diff4, d_diff), (d_spec4, d_spec)):
            _lib.check(lib.ss_env_grad_merge(src.numel() // 4, _lib.ptr(src), _lib.ptr(dst), _lib.stream_ptr()),
                       "ss_env_grad_merge")
        _, g_env = env.env_gradient(d_diff, d_spec)
    g_bg = (g_rgb * (1.0 - result.alpha)[..., None]).sum(dim=(0, 1))
    return BackwardResult(centers=g["centers"], quats=g["quats"], log_scales=g["log_scales"],
                          albedo_raw=g["albedo_raw"], metallic_raw=g["metallic_raw"],
                          roughness_raw=g["roughness_raw"], colors=g["colors"], env_base_log=g_env,
                          background=g_bg, ss_grad=g["ss_grad"], touched=g["touched"] > 0,
                          cons_loss=float(cons.item()), touch_count=g["touched"], d_diffuse=d_diff,
                          d_specular=d_spec)
