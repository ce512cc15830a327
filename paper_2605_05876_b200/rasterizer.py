"""render() / bin_and_sort() API (mirror of surfsplat.rasterizer, rasterizer.py:36-431).

render() = fused preprocess+shade kernel -> device binning + per-tile sort ->
tile-CTA forward rasteriser.  The result keeps the device state the backward
needs (records, source-indexed pair list) next to the reference-shaped
fields (compacted ProjectedSurfels, int64 tile_offsets, compacted pair_rec).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .preprocess import PreprocessOptions, ProjectedSurfels, ViewState, compact, run_preprocess

TILE = 16
K_MAX = 16
GAMMA = 2.0 * np.pi


@dataclass
class RenderOptions:
    background: tuple = (0.0, 0.0, 0.0)
    depth_mode: str = "interval"
    gamma: float = GAMMA
    k_max: int = K_MAX
    tile: int = TILE
    workers: int | None = None      # accepted for API parity; the GPU ignores it
    mip_enabled: bool = True
    mip_sigma: float = 0.1
    r_cut: float = 3.0
    dtype: type = np.float32
    shade: str = "ibl"
    collect_stacks: bool = False
    with_cover_counts: bool = False

    def preprocess_options(self):
        return PreprocessOptions(r_cut=self.r_cut, mip_enabled=self.mip_enabled, mip_sigma=self.mip_sigma)

    def validate(self):
        if self.depth_mode != "interval":
            raise ValueError(f"depth_mode {self.depth_mode!r}: the B200 path implements 'interval' only "
                             "(the ternary modes are forward-only ablations in the reference)")
        if np.dtype(self.dtype) != np.float32:
            raise ValueError("the B200 path computes in float32 (dtype=np.float32)")
        if abs(float(self.gamma) - GAMMA) > 1e-12:
            raise ValueError("only the default coverage rate gamma = 2*pi is implemented")
        if not 1 <= int(self.k_max) <= _lib.KMAX_CAP:
            raise ValueError(f"k_max must be in [1, {_lib.KMAX_CAP}]")
        if int(self.tile) not in (8, 16):
            raise ValueError("tile must be 8 or 16 (one 8x4-pixel warp block per tile quadrant)")


@dataclass
class RenderResult:
    rgb: torch.Tensor
    alpha: torch.Tensor
    depth: torch.Tensor
    nlayers: torch.Tensor
    stats: dict
    proj: ProjectedSurfels
    colors: torch.Tensor
    tile_offsets: torch.Tensor
    pair_rec: torch.Tensor
    options: RenderOptions
    camera: object
    shading_ctx: object = None
    color_source: str = "explicit"
    cover_counts: torch.Tensor | None = None
    stacks: dict | None = None
    state: ViewState | None = None          # source-indexed device state for the backward
    pair_src: torch.Tensor | None = None    # pair list in source indices
    tile_offsets32: torch.Tensor | None = None
    env: object = None


def bin_state(state: ViewState):
    """Device binning of a preprocessed view.  Returns (tile_offsets int32,
    pair list in source indices int32).  One host read of the pair total."""
    lib = _lib.load()
    dev = state.records.device
    total = int(state.tile_counts.sum().item())
    offsets = torch.empty(state.ntiles + 1, device=dev, dtype=torch.int32)
    cursors = torch.empty(state.ntiles, device=dev, dtype=torch.int32)
    keys = torch.empty(max(total, 1), device=dev, dtype=torch.int64)
    pair = torch.empty(max(total, 1), device=dev, dtype=torch.int32)
    rects = torch.empty((max(total, 1), 2), device=dev, dtype=torch.int32)
    rc = lib.ss_bin_sort(len(state.cull), _lib.ptr(state.bininfo), _lib.ptr(state.cull), state.width, state.height,
                         state.tile, _lib.ptr(state.tile_counts), _lib.ptr(offsets), _lib.ptr(cursors), _lib.ptr(keys),
                         _lib.ptr(pair), _lib.ptr(rects), total, _lib.ptr(state.flags), None, _lib.stream_ptr())
    _lib.check(rc, "ss_bin_sort")
    state.pair_rect = rects
    return offsets, pair[:total]


def _compact_index(cull):
    keep = (cull == 0)
    rank = torch.cumsum(keep.to(torch.int32), 0, dtype=torch.int32) - 1
    return keep, rank


def pack_projected(proj: ProjectedSurfels, tile=TILE, n_source=None, colors=None, cull=None):
    """ViewState of a compacted ProjectedSurfels (csrc ss_pack_records):
    records indexed by proj.source_index in a cloud of n_source rows (or by
    the compacted row itself when n_source is None), colours per source row,
    culled rows from proj.cull_code."""
    lib = _lib.load()
    dev = proj.t1.device
    k = len(proj)
    by_source = n_source is not None
    n = int(n_source) if by_source else k
    W, H = int(proj.width), int(proj.height)
    ntiles = ((W + tile - 1) // tile) * ((H + tile - 1) // tile)
    records = torch.zeros((n, _lib.REC_FLOATS), device=dev, dtype=torch.float32)
    bininfo = torch.zeros((n, 4), device=dev, dtype=torch.int32)
    tile_counts = torch.zeros(ntiles, device=dev, dtype=torch.int32)
    if cull is None:
        cull = proj.cull_code.to(torch.int8).contiguous() if by_source else torch.zeros(n, device=dev, dtype=torch.int8)
    f32 = lambda t: torch.as_tensor(t, device=dev).to(torch.float32).contiguous()
    src = torch.as_tensor(proj.source_index, device=dev).to(torch.int32).contiguous() if by_source else None
    cols = None if colors is None else f32(colors)
    rc = lib.ss_pack_records(k, _lib.ptr(f32(proj.t1)), _lib.ptr(f32(proj.t2)), _lib.ptr(f32(proj.t4)),
                             _lib.ptr(f32(proj.sinv)), _lib.ptr(f32(proj.n_f)), _lib.ptr(f32(proj.view_z)),
                             _lib.ptr(f32(proj.eps_z)),
                             _lib.ptr(torch.as_tensor(proj.rect, device=dev).to(torch.int32).contiguous()),
                             _lib.ptr(src), _lib.ptr(cols), W, H, int(tile), _lib.ptr(records), _lib.ptr(bininfo),
                             _lib.ptr(tile_counts), _lib.stream_ptr())
    _lib.check(rc, "ss_pack_records")
    flags = torch.zeros(4, device=dev, dtype=torch.int32)
    return ViewState(records, cull, tile_counts, flags, W, H, int(tile), proj.options, _lib.SS_COLOR_EXPLICIT,
                     {}, bininfo=bininfo)


def bin_and_sort(proj_or_state, tile=TILE):
    """rasterizer.py:92-116 contract: (tile_offsets int64 (T+1,), pair_rec int32
    (P,) in compacted record indices, ntx, nty).  Takes the reference's
    ProjectedSurfels (preprocess()'s output) or the ViewState of a render;
    the binning itself always runs on the device."""
    st = proj_or_state
    if isinstance(st, ProjectedSurfels):
        st = pack_projected(st, tile=tile)
        offsets, pair = bin_state(st)
        return offsets.to(torch.int64), pair.clone(), st.ntx, st.ntiles // st.ntx
    if not isinstance(st, ViewState):
        raise TypeError("bin_and_sort takes a ProjectedSurfels or the ViewState of run_preprocess/render")
    if int(tile) != st.tile:
        raise ValueError(f"the ViewState was binned for tile={st.tile}")
    offsets, pair = bin_state(st)
    _, rank = _compact_index(st.cull)
    return offsets.to(torch.int64), rank[pair.long()], st.ntx, st.ntiles // st.ntx


def render(cloud, camera, options: RenderOptions | None = None, env=None, colors=None,
           proj=None) -> RenderResult:
    """rasterizer.py:331-431.  Colours: explicit > IBL (env and shade='ibl') > albedo."""
    opt = options or RenderOptions()
    opt.validate()
    lib = _lib.load()
    if colors is not None:
        source, src_name = _lib.SS_COLOR_EXPLICIT, "explicit"
    elif env is not None and opt.shade == "ibl":
        source, src_name = _lib.SS_COLOR_IBL, "ibl"
    else:
        source, src_name = _lib.SS_COLOR_ALBEDO, "albedo"
    state = run_preprocess(cloud, camera, opt.preprocess_options(), source, colors=colors, env=env,
                           tile=int(opt.tile), want_aux=True)
    if proj is not None:
        # proj= reuse (rasterizer.py:338-339): rasterise the GIVEN projection;
        # the preprocess pass above only supplied the colours (explicit /
        # shaded / albedo per source surfel) and the shading context.  The
        # backward's per-surfel chain recomputes the projection from the
        # cloud, so proj must be this cloud's projection for this camera
        # (as preprocess() returns it) for gradients to be meaningful.
        if int(proj.width) != int(camera.width) or int(proj.height) != int(camera.height):
            raise ValueError("proj was computed for a different image size")
        if len(proj.cull_code) != len(cloud):
            raise ValueError("proj was computed for a different cloud size")
        packed = pack_projected(proj, tile=int(opt.tile), n_source=len(cloud), colors=state.aux["colors"])
        packed.aux, packed.color_source, packed.flags = state.aux, source, state.flags
        state = packed
    offsets, pair_src = bin_state(state)
    flags = state.flags.cpu()
    if int(flags[0]):
        raise ValueError("zero-norm quaternion")
    if int(flags[1]):
        raise ValueError("non-finite surfel colors")
    dev = state.records.device
    H, W = int(camera.height), int(camera.width)
    K = int(opt.k_max)
    rgb = torch.empty((H, W, 3), device=dev, dtype=torch.float32)
    alpha = torch.empty((H, W), device=dev, dtype=torch.float32)
    depth = torch.empty((H, W), device=dev, dtype=torch.float32)
    nlayers = torch.empty((H, W), device=dev, dtype=torch.int32)
    P = pair_src.shape[0]
    pair_cover = torch.zeros(max(P, 1), device=dev, dtype=torch.int32) if opt.with_cover_counts else None
    stacks = None
    st_struct = None
    if opt.collect_stacks:
        z = lambda *s: torch.zeros(s, device=dev, dtype=torch.float32)
        stacks = {"weight_sum": z(H, W, K), "color_sum": z(H, W, K, 3), "depth_sum": z(H, W, K),
                  "depth_sq_sum": z(H, W, K), "member_count": torch.zeros((H, W, K), device=dev, dtype=torch.int32)}
        st_struct = _lib.SsStacks(*(_lib.ptr(stacks[k]) for k in ("weight_sum", "color_sum", "depth_sum",
                                                                   "depth_sq_sum", "member_count")))
    discarded = torch.zeros(1, device=dev, dtype=torch.int64)
    bgp, _keep = _lib.fvec(opt.background)
    rc = lib.ss_raster_forward(W, H, int(opt.tile), _lib.ptr(offsets), _lib.ptr(pair_src), _lib.ptr(state.pair_rect),
                               _lib.ptr(state.records),
                               bgp, K, _lib.ptr(rgb), _lib.ptr(alpha), _lib.ptr(depth), _lib.ptr(nlayers),
                               _lib.ptr(pair_cover), ctypes.byref(st_struct) if st_struct is not None else None,
                               _lib.ptr(discarded), _lib.stream_ptr())
    _lib.check(rc, "ss_raster_forward")
    proj_c = compact(state) if proj is None else proj
    keep, rank = _compact_index(state.cull)
    cover_counts = None
    if opt.with_cover_counts:
        cover_counts = torch.zeros(len(cloud), device=dev, dtype=torch.int64)
        cover_counts.index_add_(0, pair_src.long(), pair_cover[:P].long())
    codes = torch.bincount(state.cull.long(), minlength=5).cpu().numpy()
    stats = {"surfels_in": len(cloud), "surfels_rasterized": int(len(proj_c)),
             "culled_nonfinite": int(codes[1]), "culled_behind": int(codes[2]),
             "culled_near_plane": int(codes[3]), "culled_offscreen": int(codes[4]),
             "pairs": int(P), "discarded_overflow": int(discarded.item()), "workers": 1}
    return RenderResult(rgb=rgb, alpha=alpha, depth=depth, nlayers=nlayers, stats=stats, proj=proj_c,
                        colors=state.aux["colors"], tile_offsets=offsets.to(torch.int64),
                        pair_rec=rank[pair_src.long()], options=opt, camera=camera,
                        shading_ctx=state.aux["cells"] if source == _lib.SS_COLOR_IBL else None,
                        color_source=src_name, cover_counts=cover_counts, stacks=stacks, state=state,
                        pair_src=pair_src, tile_offsets32=offsets, env=env)
