"""ctypes binding of libss_b200.so (include/ss_abi.h).

This is the only place the host mirror touches native code.  It fails loudly:
there is no CPU path, so a missing library or a missing CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libss_b200.so")

SS_OK, SS_ERR_INVALID, SS_ERR_CUDA = 0, 1, 2
SS_COLOR_EXPLICIT, SS_COLOR_IBL, SS_COLOR_ALBEDO, SS_COLOR_IBL_F32 = 0, 1, 2, 3
REC_FLOATS = 24
ACC_FLOATS = 20
ACC64_WIDTH = 18
KMAX_CAP = 16

c_p = ctypes.c_void_p


class SsCamera(ctypes.Structure):
    _fields_ = [("view", ctypes.c_double * 16), ("proj", ctypes.c_double * 16),
                ("width", ctypes.c_int), ("height", ctypes.c_int)]


class SsCloud(ctypes.Structure):
    _fields_ = [("centers", c_p), ("quats", c_p), ("log_scales", c_p), ("albedo_raw", c_p),
                ("metallic_raw", c_p), ("roughness_raw", c_p), ("n", ctypes.c_int)]


class SsEnv(ctypes.Structure):
    _fields_ = [("diffuse", c_p), ("specular", c_p), ("lut", c_p), ("he", ctypes.c_int),
                ("we", ctypes.c_int), ("levels", ctypes.c_int), ("lut_res", ctypes.c_int),
                ("diffuse4", c_p), ("specular4", c_p), ("diffuse64", c_p), ("specular64", c_p)]


class SsPreprocessOpts(ctypes.Structure):
    _fields_ = [("r_cut", ctypes.c_float), ("mip_sigma", ctypes.c_float),
                ("mip_enabled", ctypes.c_int), ("tile", ctypes.c_int)]


class SsProjAux(ctypes.Structure):
    _fields_ = [("c_cam", c_p), ("tu_cam", c_p), ("tv_cam", c_p), ("eps_z", c_p),
                ("center_ndc", c_p), ("jac", c_p), ("jac_ok", c_p), ("colors", c_p), ("cells", c_p),
                ("cells_packed", c_p)]


class SsStacks(ctypes.Structure):
    _fields_ = [("w", c_p), ("c", c_p), ("z", c_p), ("z2", c_p), ("n", c_p)]


class SsEnvOps(ctypes.Structure):
    _fields_ = [("rowsum", c_p), ("khat", c_p), ("row_ptr", c_p), ("col", c_p), ("rval", c_p), ("col_ptr", c_p),
                ("row", c_p), ("cval", c_p), ("work", c_p)]


class SsGrads(ctypes.Structure):
    _fields_ = [("centers", c_p), ("quats", c_p), ("log_scales", c_p), ("albedo_raw", c_p),
                ("metallic_raw", c_p), ("roughness_raw", c_p), ("colors", c_p), ("ss_grad", c_p),
                ("touched", c_p), ("d_diffuse", c_p), ("d_specular", c_p), ("d_diffuse4", c_p),
                ("d_specular4", c_p), ("view_count", c_p)]


_lib = None

_SIGNATURES = {
    "ss_preprocess": [c_p, c_p, c_p, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_preprocess_prepared": [c_p, c_p, c_p, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_surfel_prepass_bytes": [ctypes.c_int],
    "ss_adam_multi_master": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_double,
                             ctypes.c_double, ctypes.c_double, c_p],
    "ss_surfel_prepass": [c_p, c_p, c_p, c_p],
    "ss_pack_records": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_int, ctypes.c_int,
                        ctypes.c_int, c_p, c_p, c_p, c_p],
    "ss_bin_sort": [ctypes.c_int, c_p, c_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p,
                    c_p, c_p, c_p, ctypes.c_int64, c_p, c_p, c_p],
    "ss_raster_forward": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, ctypes.POINTER(ctypes.c_float),
                          ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_raster_backward": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p,
                           ctypes.POINTER(ctypes.c_float), ctypes.c_int, c_p, c_p, ctypes.c_float, c_p, c_p, c_p],
    "ss_chain_backward": [c_p, c_p, c_p, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_chain_backward_prepared": [c_p, c_p, c_p, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_diffuse_scatter": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p],
    "ss_brdf_lut": [ctypes.c_int, ctypes.c_int, c_p, c_p],
    "ss_env_khat_words": [ctypes.c_int, ctypes.c_int],
    "ss_env_khat": [ctypes.c_int, ctypes.c_int, c_p, c_p],
    "ss_env_rowsums": [ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p],
    "ss_env_refresh": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p,
                       c_p],
    "ss_env_refresh64": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p,
                         c_p, c_p],
    "ss_env_adjoint": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_spec_op_count": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p],
    "ss_spec_op_fill": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p],
    "ss_spec_apply": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_spec_apply_t": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_adam_step": [ctypes.c_int64, c_p, c_p, c_p, c_p, ctypes.c_int, ctypes.c_float, ctypes.c_float,
                     ctypes.c_float, ctypes.c_float, c_p],
    "ss_adam_step_f64": [ctypes.c_int64, c_p, c_p, c_p, c_p, ctypes.c_int, ctypes.c_float, ctypes.c_float,
                         ctypes.c_float, ctypes.c_float, c_p],
    "ss_adam_multi_f64": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_float, ctypes.c_float,
                          ctypes.c_float, c_p],
    "ss_normalize_quats": [ctypes.c_int, c_p, c_p],
    "ss_env_grad_merge": [ctypes.c_int64, c_p, c_p, c_p],
    "ss_adam_multi": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_float, ctypes.c_float,
                      ctypes.c_float, c_p],
    "ss_grid_cells": [ctypes.c_int, c_p, ctypes.POINTER(ctypes.c_float), ctypes.c_float, ctypes.c_int, c_p, c_p],
    "ss_isolation": [ctypes.c_int, c_p, c_p, c_p, c_p, ctypes.POINTER(ctypes.c_float), ctypes.c_float,
                     ctypes.c_int, c_p, c_p],
    "ss_train_forward": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, ctypes.POINTER(ctypes.c_float),
                         ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_train_coefs": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, ctypes.POINTER(ctypes.c_float),
                       c_p],
    "ss_train_forward_zstats": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, ctypes.c_int,
                                c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_train_coefs_cons": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p,
                            ctypes.c_double, c_p, c_p],
    "ss_train_backward_records_cons": [ctypes.c_int, c_p, c_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p,
                                       c_p, c_p, c_p, c_p, c_p],
    "ss_train_backward_scratch_words": [ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "ss_train_backward_records": [ctypes.c_int, c_p, c_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p,
                                  c_p, c_p, c_p, c_p],
    "ss_photometric_workspace": [ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "ss_photometric_loss": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, ctypes.c_int, ctypes.c_double, c_p, c_p,
                            c_p, c_p, c_p],
    "ss_tone_map": [ctypes.c_int64, c_p, ctypes.c_int, c_p, c_p],
    "ss_tone_map_backward": [ctypes.c_int64, c_p, ctypes.c_int, c_p, c_p, c_p],
    "ss_silhouette_loss": [ctypes.c_int64, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_knn_oriented": [ctypes.c_int, c_p, c_p, c_p, c_p, ctypes.POINTER(ctypes.c_float), ctypes.c_float, ctypes.c_int,
                        ctypes.c_int, c_p, c_p, c_p],
    "ss_normal_consistency": [ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_debug_set_fwd_timing": [c_p],
    "ss_debug_set_bwd_timing": [c_p],
    "ss_debug_cover_check": [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_cell_grid_words": [ctypes.c_int, ctypes.c_int],
    "ss_knn_workspace_bytes": [ctypes.c_int],
    "ss_cell_grid_build": [ctypes.c_int, c_p, ctypes.c_int, c_p, c_p],
    "ss_knn_dense": [ctypes.c_int, c_p, c_p, c_p, ctypes.c_int, c_p, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p, c_p],
    "ss_isolation_dense": [ctypes.c_int, c_p, c_p, c_p, ctypes.c_int, c_p, c_p],
    "ss_grid_fit": [ctypes.c_int, c_p, c_p, c_p, c_p],
    "ss_grid_cells_d": [ctypes.c_int, c_p, c_p, c_p, c_p],
    "ss_isolation_d": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_refine_workspace_bytes": [ctypes.c_int],
    "ss_refine_plan": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_int64, ctypes.c_double,
                       ctypes.c_double, c_p, c_p, c_p, c_p, c_p],
    "ss_refine_apply": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "ss_split_children": [ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_int64, ctypes.c_int64, c_p],
}

EXPORTED = [k for k in _SIGNATURES] + ["ss_last_error", "ss_version"]


def load(require_cuda=True):
    """Load the library (does not need a GPU); with require_cuda, also insist
    on a CUDA device since every entry point launches kernels."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libss_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, argt in _SIGNATURES.items():
            fn = getattr(lib, name)
            if argt is not None:
                fn.argtypes = argt
            fn.restype = ctypes.c_int
        lib.ss_photometric_workspace.restype = ctypes.c_size_t
        lib.ss_train_backward_scratch_words.restype = ctypes.c_size_t
        lib.ss_env_khat_words.restype = ctypes.c_size_t
        lib.ss_refine_workspace_bytes.restype = ctypes.c_size_t
        lib.ss_cell_grid_words.restype = ctypes.c_size_t
        lib.ss_surfel_prepass_bytes.restype = ctypes.c_size_t
        lib.ss_knn_workspace_bytes.restype = ctypes.c_size_t
        lib.ss_last_error.restype = ctypes.c_char_p
        lib.ss_version.restype = ctypes.c_int
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("paper_2605_05876_b200 needs a CUDA (sm_100a) device; there is no CPU path")
    return _lib


def check(rc, what):
    if rc == SS_OK:
        return
    if rc == SS_ERR_INVALID:
        raise ValueError(f"{what}: invalid argument")
    msg = _lib.ss_last_error().decode() if _lib is not None else "?"
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def ptr(t):
    """Device pointer of a contiguous tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return c_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_p(s.cuda_stream)


def fvec(vals):
    arr = (ctypes.c_float * len(vals))(*[float(v) for v in vals])
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_float)), arr


def make_camera(cam):
    c = SsCamera()
    v = np.ascontiguousarray(cam.view, dtype=np.float64).reshape(16)
    p = np.ascontiguousarray(cam.proj, dtype=np.float64).reshape(16)
    for k in range(16):
        c.view[k] = float(v[k])
        c.proj[k] = float(p[k])
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def make_cloud(cloud):
    return SsCloud(ptr(cloud.centers), ptr(cloud.quats), ptr(cloud.log_scales), ptr(cloud.albedo_raw),
                   ptr(cloud.metallic_raw), ptr(cloud.roughness_raw), len(cloud))


def make_env(env):
    if env is None:
        return None
    he, we = env.shape
    return SsEnv(ptr(env.diffuse), ptr(env.specular), ptr(env.lut), he, we, env.levels, env.lut.shape[0],
                 ptr(getattr(env, "diffuse4", None)), ptr(getattr(env, "specular4", None)),
                 ptr(getattr(env, "diffuse64", None)), ptr(getattr(env, "specular64", None)))


def cell_grid(centers, n, dim=None):
    """Dense cell grid over `centers` (ss_cell_grid_build): (words, dim).
    dim ~ sqrt(n / 24) so a surface sampling puts about ten surfels in each
    occupied cell (<= 512: at most a 1 GB table; 4M surfels take dim 408)."""
    if dim is None:
        dim = int(min(512, max(1, round((max(n, 1) / 24.0) ** 0.5))))
    lib = load()
    words = torch.empty(int(lib.ss_cell_grid_words(n, dim)), device=centers.device, dtype=torch.int32)
    check(lib.ss_cell_grid_build(n, ptr(centers), dim, ptr(words), stream_ptr()), "ss_cell_grid_build")
    return words, dim
