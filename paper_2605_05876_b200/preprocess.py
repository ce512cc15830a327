"""Per-view preprocessing API (mirror of surfsplat.preprocess, preprocess.py:30-309).

run_preprocess() launches the fused projection/filter/bounding/shading/tile-
count kernel (csrc/preprocess.cu) and returns the raw per-source-surfel
state; preprocess() additionally compacts the kept rows into a
ProjectedSurfels like the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib

R_CUT = 3.0
DENOM_EPS = 1e-9
VIEW_Z_EPS = 1e-4
CULL_NONE, CULL_NONFINITE, CULL_BEHIND, CULL_NEAR_PLANE, CULL_OFFSCREEN = 0, 1, 2, 3, 4


@dataclass
class PreprocessOptions:
    r_cut: float = R_CUT
    mip_enabled: bool = True
    mip_sigma: float = 0.1
    dtype: type = None


@dataclass
class ViewState:
    """Device state of one projected view (source-indexed)."""
    records: torch.Tensor      # (N, 24) float32, see SsRecord
    cull: torch.Tensor         # (N,) int8
    tile_counts: torch.Tensor  # (ntiles,) int32
    flags: torch.Tensor        # (4,) int32
    width: int
    height: int
    tile: int
    options: PreprocessOptions
    color_source: int
    aux: dict = field(default_factory=dict)
    pair_rect: torch.Tensor | None = None  # (P, 2) int32 packed rects in pair order (after binning)
    bininfo: torch.Tensor | None = None    # (N, 4) int32 binning input (packed rect, z_start key)

    @property
    def ntx(self):
        return (self.width + self.tile - 1) // self.tile

    @property
    def ntiles(self):
        return self.ntx * ((self.height + self.tile - 1) // self.tile)


def make_opts(options, tile=16):
    return _lib.SsPreprocessOpts(float(options.r_cut), float(options.mip_sigma), int(bool(options.mip_enabled)), int(tile))


def run_preprocess(cloud, camera, options, color_source, colors=None, env=None, tile=16, want_aux=False,
                   records=None, cull=None, tile_counts=None, flags=None, bininfo=None):
    lib = _lib.load()
    n = len(cloud)
    dev = cloud.centers.device
    W, H = int(camera.width), int(camera.height)
    ntiles = ((W + tile - 1) // tile) * ((H + tile - 1) // tile)
    records = torch.empty((n, _lib.REC_FLOATS), device=dev, dtype=torch.float32) if records is None else records
    cull = torch.empty(n, device=dev, dtype=torch.int8) if cull is None else cull
    bininfo = torch.empty((n, 4), device=dev, dtype=torch.int32) if bininfo is None else bininfo
    if tile_counts is None:
        tile_counts = torch.zeros(ntiles, device=dev, dtype=torch.int32)
    else:
        tile_counts.zero_()
    if flags is None:
        flags = torch.zeros(4, device=dev, dtype=torch.int32)
    else:
        flags.zero_()
    aux = {}
    auxs = None
    if want_aux:
        f = lambda *s: torch.zeros(s, device=dev, dtype=torch.float32)
        aux = {"c_cam": f(n, 3), "tu_cam": f(n, 3), "tv_cam": f(n, 3), "eps_z": f(n), "center_ndc": f(n, 2),
               "jac": f(n, 2, 2), "jac_ok": torch.zeros(n, device=dev, dtype=torch.uint8), "colors": f(n, 3),
               "cells": torch.zeros((n, 15), device=dev, dtype=torch.int32),
               "cells_packed": torch.zeros((n, 4), device=dev, dtype=torch.int32)}
        auxs = _lib.SsProjAux(*(_lib.ptr(aux[k]) for k in ("c_cam", "tu_cam", "tv_cam", "eps_z", "center_ndc",
                                                            "jac", "jac_ok", "colors", "cells", "cells_packed")))
    cam = _lib.make_camera(camera)
    cl = _lib.make_cloud(cloud)
    opt = make_opts(options, tile)
    envs = _lib.make_env(env)
    if colors is not None:
        colors = torch.as_tensor(colors, device=dev, dtype=torch.float32).contiguous()
    rc = lib.ss_preprocess(ctypes_ref(cl), ctypes_ref(cam), ctypes_ref(opt), int(color_source), _lib.ptr(colors),
                           ctypes_ref(envs) if envs is not None else None, _lib.ptr(records), _lib.ptr(cull), None,
                           _lib.ptr(tile_counts), _lib.ptr(bininfo), ctypes_ref(auxs) if auxs is not None else None,
                           _lib.ptr(flags), _lib.stream_ptr())
    _lib.check(rc, "ss_preprocess")
    return ViewState(records, cull, tile_counts, flags, W, H, tile, options, color_source, aux, bininfo=bininfo)


def ctypes_ref(s):
    import ctypes
    return ctypes.byref(s)


@dataclass
class ProjectedSurfels:
    """Culled, compacted per-view records (preprocess.py:195-228), device tensors."""
    t1: torch.Tensor
    t2: torch.Tensor
    t4: torch.Tensor
    view_z: torch.Tensor
    eps_z: torch.Tensor
    sinv: torch.Tensor
    n_f: torch.Tensor
    center_ndc: torch.Tensor
    jac: torch.Tensor
    jac_ok: torch.Tensor
    rect: torch.Tensor
    source_index: torch.Tensor
    c_cam: torch.Tensor
    tu_cam: torch.Tensor
    tv_cam: torch.Tensor
    cull_code: torch.Tensor
    width: int
    height: int
    options: PreprocessOptions

    def __len__(self):
        return self.view_z.shape[0]

    @property
    def z_start(self):
        return self.view_z - self.eps_z

    @property
    def z_end(self):
        return self.view_z + self.eps_z


def compact(state: ViewState) -> ProjectedSurfels:
    keep = torch.nonzero(state.cull == 0).flatten()
    r = state.records[keep]
    a = state.aux
    rect = r[:, 20:24].contiguous().view(torch.int32)
    return ProjectedSurfels(
        t1=r[:, 0:3].contiguous(), t2=r[:, 3:6].contiguous(), t4=r[:, 6:9].contiguous(),
        view_z=r[:, 13].contiguous(), eps_z=a["eps_z"][keep], sinv=r[:, 9:12].contiguous(),
        n_f=r[:, 12].contiguous(), center_ndc=a["center_ndc"][keep], jac=a["jac"][keep],
        jac_ok=a["jac_ok"][keep].bool(), rect=rect, source_index=keep.to(torch.int32),
        c_cam=a["c_cam"][keep], tu_cam=a["tu_cam"][keep], tv_cam=a["tv_cam"][keep],
        cull_code=state.cull.clone(), width=state.width, height=state.height, options=state.options)


def preprocess(cloud, camera, options: PreprocessOptions | None = None) -> ProjectedSurfels:
    """preprocess.py:231-309: project, filter, bound and cull one view."""
    opt = options or PreprocessOptions()
    st = run_preprocess(cloud, camera, opt, color_source=_lib.SS_COLOR_ALBEDO, want_aux=True)
    if int(st.flags[0].item()):
        raise ValueError("zero-norm quaternion")
    return compact(st)
