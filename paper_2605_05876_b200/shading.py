"""Environment light and split-sum shading API (mirror of surfsplat.shading).

EnvironmentLight keeps the learnable log radiance (He, We, 3) and the derived
maps (irradiance, GGX roughness chain, BRDF LUT) as float32 CUDA tensors.
refresh() and env_gradient() run the on-the-fly operator kernels of
csrc/env.cu (shading.py:369-394); nothing T x T is ever materialised.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

DEFAULT_ENV_SHAPE = (16, 32)
DEFAULT_LEVELS = 6
DEFAULT_LUT_RES = 64
DEFAULT_LUT_SAMPLES = 128
DEFAULT_SPEC_SAMPLES = 128

_LUT_CACHE = {}
_OPS_CACHE = {}


def brdf_lut(res=DEFAULT_LUT_RES, samples=DEFAULT_LUT_SAMPLES):
    """(res, res, 2) float32 device LUT, row = roughness (shading.py:118-156)."""
    key = (res, samples, torch.cuda.current_device())
    if key not in _LUT_CACHE:
        lib = _lib.load()
        lut = torch.empty((res, res, 2), device="cuda", dtype=torch.float32)
        _lib.check(lib.ss_brdf_lut(res, samples, _lib.ptr(lut), _lib.stream_ptr()), "ss_brdf_lut")
        _LUT_CACHE[key] = lut
    return _LUT_CACHE[key]


class EnvOps:
    """The prefilter operators of one env shape on one device, as the
    caller-owned buffers ss_env_refresh / ss_env_adjoint take (SsEnvOps):
    diffuse row sums, the diffuse kernel's spectrum (K^, float64), the
    sparse specular operator (CSR) and its per-level transpose (CSC), and the
    float64 work area.  Built once per (He, We, L, samples, device) -- the
    reference's build_diffuse_operator / build_specular_operator
    (shading.py:275-331) without ever forming the dense T x T matrices."""

    def __init__(self, he, we, levels, samples):
        lib = _lib.load()
        dev = torch.device("cuda", torch.cuda.current_device())
        s = _lib.stream_ptr()
        T = he * we
        self.work = torch.empty(3 * T, device=dev, dtype=torch.float64)
        nk = int(lib.ss_env_khat_words(he, we))
        self.khat = None
        if nk:
            self.khat = torch.empty(nk, device=dev, dtype=torch.float64)
            _lib.check(lib.ss_env_khat(he, we, _lib.ptr(self.khat), s), "ss_env_khat")
        self.rowsum = torch.empty(T, device=dev, dtype=torch.float64)
        _lib.check(lib.ss_env_rowsums(he, we, _lib.ptr(self.khat), _lib.ptr(self.rowsum), _lib.ptr(self.work), s),
                   "ss_env_rowsums")
        self.spec = None
        if levels >= 2:
            nrows = (levels - 1) * T
            nnz = torch.empty(nrows, device=dev, dtype=torch.int32)
            _lib.check(lib.ss_spec_op_count(he, we, levels, samples, _lib.ptr(nnz), s), "ss_spec_op_count")
            row_ptr = torch.zeros(nrows + 1, device=dev, dtype=torch.int64)
            row_ptr[1:] = torch.cumsum(nnz.to(torch.int64), 0)
            total = int(row_ptr[-1].item())
            col = torch.empty(total, device=dev, dtype=torch.int32)
            rval = torch.empty(total, device=dev, dtype=torch.float64)
            _lib.check(lib.ss_spec_op_fill(he, we, levels, samples, _lib.ptr(row_ptr), _lib.ptr(col), _lib.ptr(rval),
                                           s), "ss_spec_op_fill")
            rows = torch.repeat_interleave(torch.arange(nrows, device=dev, dtype=torch.int64), nnz.to(torch.int64))
            key_c = (rows // T) * T + col.to(torch.int64)
            order = torch.sort(key_c, stable=True).indices
            row_t = (rows[order] % T).to(torch.int32).contiguous()
            cval = rval[order].contiguous()
            col_ptr = torch.zeros(nrows + 1, device=dev, dtype=torch.int64)
            col_ptr[1:] = torch.cumsum(torch.bincount(key_c, minlength=nrows), 0)
            self.spec = (row_ptr, col, rval, col_ptr, row_t, cval)
        sp = self.spec or (None,) * 6
        self.struct = _lib.SsEnvOps(_lib.ptr(self.rowsum), _lib.ptr(self.khat), *(_lib.ptr(t) for t in sp),
                                    _lib.ptr(self.work))

    def ref(self):
        return ctypes.byref(self.struct)


def env_ops(he, we, levels=DEFAULT_LEVELS, samples=DEFAULT_SPEC_SAMPLES):
    key = (he, we, levels, samples, torch.cuda.current_device())
    if key not in _OPS_CACHE:
        _OPS_CACHE[key] = EnvOps(he, we, levels, samples)
    return _OPS_CACHE[key]


class EnvironmentLight:
    """Learnable lat-long environment (shading.py:334-409)."""

    def __init__(self, base_log, levels=DEFAULT_LEVELS, lut_res=DEFAULT_LUT_RES,
                 lut_samples=DEFAULT_LUT_SAMPLES, spec_samples=DEFAULT_SPEC_SAMPLES):
        t = base_log if isinstance(base_log, torch.Tensor) else torch.from_numpy(np.asarray(base_log, dtype=np.float64))
        t = t.to(device="cuda", dtype=torch.float32).contiguous()
        if t.dim() != 3 or t.shape[2] != 3 or min(t.shape[:2]) < 2:
            raise ValueError("base_log must be (He >= 2, We >= 2, 3)")
        if levels < 1:
            raise ValueError("at least one roughness level")
        self.base_log = t
        self.levels, self.lut_res, self.lut_samples, self.spec_samples = int(levels), int(lut_res), int(lut_samples), int(spec_samples)
        he, we = self.shape
        self.base = torch.empty_like(t)
        self.diffuse = torch.empty_like(t)
        self.specular = torch.empty((self.levels, he, we, 3), device="cuda", dtype=torch.float32)
        # 16-byte texels for the shading kernels' bilinear fetches
        self.diffuse4 = torch.zeros((he, we, 4), device="cuda", dtype=torch.float32)
        self.specular4 = torch.zeros((self.levels, he, we, 4), device="cuda", dtype=torch.float32)
        # the float64 maps (the reference's precision), read by the float64 shading
        self.base64 = torch.empty((he, we, 3), device="cuda", dtype=torch.float64)
        self.diffuse64 = torch.empty((he, we, 3), device="cuda", dtype=torch.float64)
        self.specular64 = torch.empty((self.levels, he, we, 3), device="cuda", dtype=torch.float64)
        self.refresh()

    @property
    def shape(self):
        return tuple(self.base_log.shape[:2])

    @property
    def lut(self):
        return brdf_lut(self.lut_res, self.lut_samples)

    def level_roughness(self):
        if self.levels == 1:
            return np.zeros(1)
        return np.arange(self.levels) / (self.levels - 1.0)

    def refresh(self, base_log64=None):
        """Derived maps from base_log (shading.py:369-379); base_log64: a float64
        master of it (Adam(master_params=True)) to refresh from instead."""
        lib = _lib.load()
        he, we = self.shape
        ops = env_ops(he, we, self.levels, self.spec_samples)
        fn, src = lib.ss_env_refresh, self.base_log
        if base_log64 is not None:
            if tuple(base_log64.shape) != tuple(self.base_log.shape) or base_log64.dtype != torch.float64:
                raise ValueError("base_log64 must be a float64 tensor shaped like base_log")
            fn, src = lib.ss_env_refresh64, base_log64
        _lib.check(fn(he, we, self.levels, self.spec_samples, _lib.ptr(src), ops.ref(),
                                      _lib.ptr(self.base), _lib.ptr(self.diffuse), _lib.ptr(self.specular),
                                      _lib.ptr(self.base64), _lib.ptr(self.diffuse64), _lib.ptr(self.specular64),
                                      _lib.stream_ptr()), "ss_env_refresh")
        self.diffuse4[..., :3].copy_(self.diffuse)
        self.specular4[..., :3].copy_(self.specular)

    def env_gradient(self, d_diffuse, d_specular):
        """Derived-map gradients -> (d_base, d_base_log) (shading.py:381-394)."""
        lib = _lib.load()
        he, we = self.shape
        f64 = dict(device="cuda", dtype=torch.float64)
        dd = torch.as_tensor(d_diffuse, **f64).contiguous() if d_diffuse is not None \
            else torch.zeros(self.base.shape, **f64)
        ds = torch.as_tensor(d_specular, **f64).contiguous() if d_specular is not None \
            else torch.zeros(self.specular.shape, **f64)
        d_base = torch.empty(self.base.shape, **f64)
        d_log = torch.empty_like(self.base)
        ops = env_ops(he, we, self.levels, self.spec_samples)
        _lib.check(lib.ss_env_adjoint(he, we, self.levels, self.spec_samples, _lib.ptr(self.base64), ops.ref(),
                                      _lib.ptr(dd), _lib.ptr(ds), _lib.ptr(d_base), _lib.ptr(d_log),
                                      _lib.stream_ptr()), "ss_env_adjoint")
        return d_base, d_log

    @staticmethod
    def uniform(value=0.5, shape=DEFAULT_ENV_SHAPE, levels=DEFAULT_LEVELS):
        return EnvironmentLight(np.log(np.full(tuple(shape) + (3,), float(value))), levels=levels)

    @staticmethod
    def from_base(base, levels=DEFAULT_LEVELS):
        return EnvironmentLight(np.log(np.maximum(np.asarray(base, dtype=np.float64), 1e-8)), levels=levels)

    def copy(self):
        return EnvironmentLight(self.base_log.clone(), self.levels, self.lut_res, self.lut_samples, self.spec_samples)


SRGB_LIN_BOUND = 0.0031308
TONE_MODES = {"ldr": 0, "hdr-loss": 1}


def _tone_mode(mode):
    if mode not in TONE_MODES:
        raise ValueError(f"unknown tone map mode {mode!r}")
    return TONE_MODES[mode]


def _f32_cuda(x):
    return torch.as_tensor(x, device="cuda", dtype=torch.float32).contiguous()


def tone_map(img, mode="ldr"):
    """shading.py:54-67 ('ldr': sRGB of the [0, 1] clamp, 'hdr-loss': sRGB of
    log1p(max(x, 0))) -- csrc/losses.cu ss_tone_map, float64 inside."""
    m = _tone_mode(mode)
    x = _f32_cuda(img)
    out = torch.empty_like(x)
    lib = _lib.load()
    _lib.check(lib.ss_tone_map(x.numel(), _lib.ptr(x), m, _lib.ptr(out), _lib.stream_ptr()), "ss_tone_map")
    return out


def tone_map_backward(img, mode, g_out):
    """shading.py:70-79: d tone_map / d img applied to an upstream gradient."""
    m = _tone_mode(mode)
    x = _f32_cuda(img)
    g = _f32_cuda(g_out)
    if g.shape != x.shape:
        raise ValueError("image shape mismatch")
    out = torch.empty_like(x)
    lib = _lib.load()
    _lib.check(lib.ss_tone_map_backward(x.numel(), _lib.ptr(x), m, _lib.ptr(g), _lib.ptr(out), _lib.stream_ptr()),
               "ss_tone_map_backward")
    return out


def shade_surfels(cloud, env, camera):
    """Per-surfel IBL colours (shading.py:447-503) via the preprocess kernel's
    shading stage.  Returns (colors (N,3) float32, cells (N,15) int32)."""
    from .preprocess import PreprocessOptions, run_preprocess
    st = run_preprocess(cloud, camera, PreprocessOptions(), color_source=_lib.SS_COLOR_IBL, env=env,
                        want_aux=True)
    return st.aux["colors"], st.aux["cells"]
