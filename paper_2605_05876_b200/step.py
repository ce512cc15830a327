"""Batched inverse-rendering step: the BASELINE "fwd+bwd view" workload.

One step = for every view of the batch: preprocess+shade, device binning and
per-tile sort, fused forward + L1 loss + per-pixel suffix recursion, pass-2
backward, per-surfel chain (accumulating into the step's gradient buffer);
then the environment adjoint once for the batch, an NCCL all-reduce of the
packed gradients when running data-parallel (views sharded across ranks,
surfels/env replicated), Adam on every parameter tensor, quaternion
renormalisation and the environment refresh.  This is the reference's
`fit` step body (train.py:188-248) with the loss of BASELINE config 0 (L1 in
linear space) and a batch of views instead of one (gradients summed over
views, the batching SURVEY.md §7 hard part 7 defines).

The views are issued asynchronously; the step reads ONE small status block
back before applying the optimiser: the binning kernel's pair-overflow flag
(all-reduced with the gradients, so every rank agrees), the pairs the
largest view needed, and the preprocess flags.  Pair buffers are sized from a
measured view (x1.5); when a later view needs more (a closer camera, scales
grown by training) the buffers grow to fit and the step's views are re-run
before any parameter changes -- a silently truncated tile list never reaches
Adam.  A zero-norm quaternion or a non-finite colour raises ValueError, as
the reference's render() does (rasterizer.py:352-353).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .adam import Adam
from .preprocess import PreprocessOptions, make_opts

PARAMS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw")
_WIDTH = {"centers": 3, "quats": 4, "log_scales": 2, "albedo_raw": 3, "metallic_raw": 1, "roughness_raw": 1}


def shard_views(n_views, world, rank):
    """Contiguous block of the step's views owned by `rank` (views split evenly;
    the first n_views % world ranks take one extra)."""
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def collectives_on(group=None):
    """Whether the step's gradients go through a collective: a process group
    with more than one rank, or any initialised group when SS_COLLECTIVES=force
    (the NCCL self-test: one rank, the same calls and stream ordering as a
    multi-GPU run)."""
    if not (dist.is_available() and dist.is_initialized()):
        return False
    return dist.get_world_size(group) > 1 or os.environ.get("SS_COLLECTIVES") == "force"


class GradPack:
    """One flat buffer holding everything the step all-reduces: the 14
    parameter channels per surfel, ss_grad, the per-surfel count of views the
    surfel covered a pixel in (`view_count`, the sum over the step's views of
    backward_image's `touched` bool, backward.py:432-441 -- what
    DensifyStats.accumulate adds per view, densify.py:35-37; exact in float32
    up to 2^24 views), the env log-radiance gradient and the loss -- a single
    collective per step."""

    def __init__(self, n, env_texels, device, dtype=torch.float32):
        sizes = [n * _WIDTH[k] for k in PARAMS] + [n, n, 3 * env_texels, 1, 1]
        # every segment starts 16-byte aligned (the chain kernel adds
        # quaternion gradients with 16-byte vector reductions)
        pad = lambda v: (v + 3) & ~3
        self.flat = torch.zeros(sum(pad(s) for s in sizes), device=device, dtype=dtype)
        views, off = [], 0
        for s in sizes:
            views.append(self.flat[off:off + s])
            off += pad(s)
        self.grads = {k: views[i].view(n, _WIDTH[k]) if _WIDTH[k] > 1 else views[i] for i, k in enumerate(PARAMS)}
        self.grads["ss_grad"] = views[len(PARAMS)]
        self.view_count = views[len(PARAMS) + 1]
        self.env = views[len(PARAMS) + 2]
        self.loss = views[len(PARAMS) + 3]
        self.status = views[len(PARAMS) + 4]  # > 0: some rank's pair buffers overflowed this step

    @property
    def touched(self):
        """Alias of view_count (per-surfel number of views touched)."""
        return self.view_count

    def zero(self):
        self.flat.zero_()

    def _bucket_split(self):
        # bucket A: the per-surfel channels (params, ss_grad, view_count) --
        # final once the last view's chain kernel ran; bucket B: env gradient,
        # loss and status -- final only after the env adjoint
        return self.env.data_ptr() - self.flat.data_ptr()

    def all_reduce_surfels(self, group=None):
        """Start the all-reduce of bucket A asynchronously (NCCL runs it on its
        own stream after the work queued so far); returns the work handle or
        None when not distributed."""
        if collectives_on(group):
            n = self._bucket_split() // self.flat.element_size()
            return dist.all_reduce(self.flat[:n], group=group, async_op=True)
        return None

    def all_reduce_rest(self, group=None):
        """All-reduce bucket B (env gradient, loss, status: ~T*3 + 2 floats)."""
        if collectives_on(group):
            n = self._bucket_split() // self.flat.element_size()
            dist.all_reduce(self.flat[n:], group=group)

    def all_reduce(self, group=None, async_op=False):
        """The whole buffer in one collective."""
        if collectives_on(group):
            return dist.all_reduce(self.flat, group=group, async_op=async_op)
        return None


class ViewBuffers:
    """Device scratch of one in-flight view (records, pair lists, per-pixel
    training planes, record accumulator).  TrainStep keeps one set per stream
    so consecutive views overlap on the GPU."""

    def __init__(self, n, W, H, tile, k_max, ntiles, device):
        f32 = dict(device=device, dtype=torch.float32)
        i32 = dict(device=device, dtype=torch.int32)
        self.records = torch.empty((n, _lib.REC_FLOATS), **f32)
        self.cull = torch.empty(n, device=device, dtype=torch.int8)
        self.bininfo = torch.empty((n, 4), **i32)
        self.tile_counts = torch.zeros(ntiles, **i32)
        self.flags = torch.zeros(4, **i32)
        self.offsets = torch.empty(ntiles + 1, **i32)
        self.cursors = torch.empty(ntiles, **i32)
        self.tile_order = torch.empty(ntiles, **i32)
        # per layer and pixel: float4 (A hi, dL/dC_raw), a float plane of A lo, a float4 plane of raw-sum lo (ss_abi.h)
        self.coef = torch.empty(9 * k_max * H * W, **f32)
        self.thr = torch.empty((k_max, H * W), **f32)
        self.pix_hdr = torch.empty((H * W, 8), **i32)
        # NDC tables, counters, area-class sort and big-rect queue of the backward
        self.pixel_ndc = torch.empty(_lib.load().ss_train_backward_scratch_words(n, W, H), **f32)
        self.acc = torch.zeros((n, _lib.ACC_FLOATS), **f32)
        # the float64 shading forward's packed branch state (SsProjAux.cells_packed)
        self.cells = torch.empty((n, 4), device=device, dtype=torch.int32)
        self.aux = _lib.SsProjAux(*([None] * 9), _lib.ptr(self.cells))
        # float64 channel rows of the big records (SS_ACC_F64)
        self.acc64 = torch.empty((n, _lib.ACC64_WIDTH), device=device, dtype=torch.float64)
        # this buffer set's share of the step loss (photometric mode): views on
        # different worker streams never read-modify-write the same scalar
        self.loss_part = torch.zeros(1, device=device, dtype=torch.float64)
        self.capacity = 0
        self.keys = self.pair = self.pair_rect = None

    def alloc_zstats(self, k_max, W, H):
        """Per-layer depth moments / penalty coefficients of the consolidation
        term (allocated on first use)."""
        if getattr(self, "zst", None) is None:
            self.zst = torch.empty((k_max, H * W, 4), device=self.coef.device, dtype=torch.float32)

    def alloc_loss(self, W, H, device):
        """Buffers of the deferred-loss step (photometric loss on the image)."""
        from .losses import ImageLoss
        f32 = dict(device=device, dtype=torch.float32)
        self.rgb = torch.empty((H, W, 3), **f32)
        self.g_rgb = torch.empty((H, W, 3), **f32)
        # the image gradient in float64 as well: the layer coefficients'
        # colour terms cancel, and a float32-rounded gradient biases them
        self.g_rgb64 = torch.empty((H, W, 3), device=device, dtype=torch.float64)
        self.alpha = torch.empty((H, W), **f32)
        self.g_alpha = torch.empty((H, W), **f32)
        self.sil = torch.zeros(1, device=device, dtype=torch.float64)
        self.sil_ws = torch.empty(2, device=device, dtype=torch.float64)
        self.imgloss = ImageLoss(H, W, 3, device)

    def alloc_pairs(self, cap):
        dev = self.records.device
        self.keys = torch.empty(cap, device=dev, dtype=torch.int64)
        self.pair = torch.empty(cap, device=dev, dtype=torch.int32)
        self.pair_rect = torch.empty((cap, 2), device=dev, dtype=torch.int32)
        self.capacity = cap


class TrainStep:
    def __init__(self, cloud, env, width, height, k_max=16, tile=16, background=(0.0, 0.0, 0.0),
                 lrs=None, pair_capacity=None, process_group=None, options=None, streams=2, loss="l1",
                 tone="hdr-loss", lambda_ssim=0.2, lambda_sil=0.1, cons_scale=0.0, surfel_capacity=None,
                 master_params=True):
        """loss="l1": the BASELINE config loss (mean |rgb - target| in linear
        space), fused into the forward kernel.  loss="photometric": the
        reference fit loss (train.py:194-206): tone_map(tone) then
        (1 - lambda_ssim) L1 + lambda_ssim (1 - SSIM) on the device, plus
        lambda_sil * silhouette when masks are given to step(), plus the
        depth-consolidation penalty with weight cons_scale (the reference's
        lambda_cons / (extent * npix) of its main phase, train.py:208-213;
        settable between steps as `ts.cons_scale`).  surfel_capacity: size
        the per-view buffers for up to this many surfels, so refine() can
        grow the cloud (up to it) without reallocating them."""
        if loss not in ("l1", "photometric"):
            raise ValueError(f"unknown loss {loss!r}")
        self.loss_mode, self.tone, self.lambda_ssim, self.lambda_sil = loss, tone, float(lambda_ssim), float(lambda_sil)
        if float(cons_scale) > 0.0 and loss != "photometric":
            raise ValueError("the consolidation penalty needs loss='photometric' (deferred coefficients)")
        self.cons_scale = float(cons_scale)
        self.lib = _lib.load()
        self.cloud, self.env = cloud, env
        self.W, self.H, self.k_max, self.tile = int(width), int(height), int(k_max), int(tile)
        self.bg = tuple(float(b) for b in background)
        self.opts = options or PreprocessOptions()
        self.pg = process_group
        self.lrs = lrs or {"centers": 1.6e-4, "quats": 1e-3, "log_scales": 5e-3, "albedo_raw": 5e-3,
                           "metallic_raw": 5e-3, "roughness_raw": 5e-3, "env_base_log": 1e-2}
        n = len(cloud)
        dev = cloud.centers.device
        self.n = n
        self.surfel_capacity = max(n, int(surfel_capacity or 0), 1)
        self.ntx = (self.W + tile - 1) // tile
        self.ntiles = self.ntx * ((self.H + tile - 1) // tile)
        self.bufs = [ViewBuffers(self.surfel_capacity, self.W, self.H, tile, self.k_max, self.ntiles, dev)
                     for _ in range(max(1, streams))]
        # the buffer sets' flag words side by side: one read-back per step
        self.flags_all = torch.zeros((len(self.bufs), 4), device=dev, dtype=torch.int32)
        for i, b in enumerate(self.bufs):
            b.flags = self.flags_all[i]
        he, we = env.shape
        for b in self.bufs:  # per-view float32 derived-map accumulators (16-byte texels)
            b.d_diff4 = torch.zeros((he, we, 4), device=dev, dtype=torch.float32)
            b.d_spec4 = torch.zeros((env.levels, he, we, 4), device=dev, dtype=torch.float32)
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(len(self.bufs))]
        if loss == "photometric":
            for b in self.bufs:
                b.alloc_loss(self.W, self.H, dev)
        he, we = env.shape
        self.T = he * we
        self.loss = torch.zeros(1, device=dev, dtype=torch.float64)
        self.d_diffuse = torch.zeros(env.base.shape, device=dev, dtype=torch.float64)
        self.d_spec = torch.zeros(env.specular.shape, device=dev, dtype=torch.float64)
        # each buffer set folds its views' derived-map sums into its own
        # float64 maps (no ordering between the worker streams); the sets are
        # summed once per step (the first set's maps are the step's own)
        for k, b in enumerate(self.bufs):
            b.d_diffuse64 = self.d_diffuse if k == 0 else torch.zeros_like(self.d_diffuse)
            b.d_spec64 = self.d_spec if k == 0 else torch.zeros_like(self.d_spec)
        self.d_base = torch.empty(env.base.shape, device=dev, dtype=torch.float64)
        # float64 master parameters like the reference's fit (train.py:168-174)
        self.adam = Adam(master_params=master_params)
        self._po = make_opts(self.opts, tile)
        self._envs = _lib.make_env(env)
        self._bind_cloud(cloud)
        self._bg = _lib.fvec(self.bg)
        self.capacity = 0
        self.regrows = 0           # times a step re-ran its views after growing the pair buffers
        if pair_capacity:
            self._alloc_pairs(pair_capacity)
        self.collect_stats = False
        self.captured_rgb = None       # a list -> the forward's image of every view is appended
        # forward colours: float64 IBL shading like render() (the step's image
        # is then bit-identical to the API path's and within 1e-4 of the
        # oracle); SS_COLOR_IBL_F32 is the float32 variant (colours within
        # ~1e-4 relative: texel coordinates at 256-texel rows carry ~1e-5
        # texel float32 rounding)
        self.color_source = _lib.SS_COLOR_IBL
        self._pairs, self._kept, self._layer_px, self._nviews = [], [], [], 0
        self.kernel_events = None      # list -> (name, start, end) CUDA events per raster launch
        self._graphs = {}              # step(graph=True): captured gradient passes by (cameras, inputs)
        self.active_streams = None     # None: all worker streams; 1: views serialised (isolated kernel timing)
        self._stage = None
        # preprocess, scan + order, scatter, tile sort x2, train fwd, ndc, area class, class scatter,
        # record bwd, big-rect bwd, big-rect finish, chain, env merge (specular; + diffuse when the
        # diffuse taps are scattered per view)
        self.launches_per_view = 14
        # prepass, diffuse scatter, env adjoint (spectral diffuse 3, specular SpMV, finish), fused
        # Adam (+ quat renorm), env refresh (exp, narrow, spectral diffuse 3, specular SpMV) --
        # the ncu launch list of profiles/r2j_launches.txt
        self.launches_per_step_fixed = 1 + 1 + 5 + 1 + 6

    # -- buffers -----------------------------------------------------------
    def _bind_cloud(self, cloud):
        """(Re)bind the per-surfel state to `cloud`: the packed gradient
        buffer (params, ss_grad, view counts, env, loss -- one all-reduce
        buffer) and the native views of both."""
        he, we = self.env.shape
        dev = cloud.centers.device
        self._graphs = {}  # captured launches hold the old cloud's pointers
        self.cloud = cloud
        self.n = len(cloud)
        if self.n > self.surfel_capacity:  # grow the per-view buffers
            self.surfel_capacity = self.n
            for b in self.bufs:
                nb = ViewBuffers(self.n, self.W, self.H, self.tile, self.k_max, self.ntiles, dev)
                for k in ("records", "cull", "bininfo", "pixel_ndc", "acc", "acc64", "cells", "aux"):
                    setattr(b, k, getattr(nb, k))
        self.pack = GradPack(self.n, self.T, dev)
        self.flat = self.pack.flat
        self.grads = self.pack.grads
        self.g_env_log = self.pack.env.view(he, we, 3)
        self.loss_f = self.pack.loss
        self.view_count = self.pack.view_count
        self._cl = _lib.make_cloud(cloud)
        # the step's view-independent per-surfel state (ss_surfel_prepass) and the
        # per-surfel diffuse-lookup upstream of its views (ss_chain_backward_prepared;
        # ss_diffuse_scatter applies the taps once per step and re-zeroes it): sized
        # for the surfel capacity, so a refinement step's rebinding does not reallocate
        cap = self.surfel_capacity
        if getattr(self, "_prepass_cap", 0) < cap:
            self._prepass = torch.empty(int(self.lib.ss_surfel_prepass_bytes(cap)), device=dev, dtype=torch.uint8)
            self._g_ld = torch.zeros(4 * cap, device=dev, dtype=torch.float32)
            self._prepass_cap = cap
        else:
            self._g_ld[:4 * self.n].zero_()
        self._prepared = False
        for b in self.bufs:
            b.gs = _lib.SsGrads(*(_lib.ptr(self.grads[k]) for k in PARAMS), None, _lib.ptr(self.grads["ss_grad"]),
                                None, _lib.ptr(b.d_diffuse64), _lib.ptr(b.d_spec64),
                                _lib.ptr(b.d_diff4), _lib.ptr(b.d_spec4), _lib.ptr(self.view_count))

    def refine(self, stats, mean_neighbor_dist, max_surfels, quantile=0.9, grad_floor=1e-8,
               outside_mask_votes=None, front_votes=None):
        """The density-aware refinement pass after a step (train.py:260-276):
        refine_topology on the device (prune, quantile threshold, budget,
        split) with the optimiser state remapped in the same pass
        (Adam.remap), then the step rebinds to the new cloud (self.cloud).
        Returns (index_map, reasons); the caller resets its DensifyStats and
        rebuilds its neighbour index, as the reference does."""
        from .densify import refine_topology
        new, index_map, reasons = refine_topology(self.cloud, stats, mean_neighbor_dist, max_surfels, quantile,
                                                  grad_floor, outside_mask_votes, front_votes, optimizer=self.adam)
        self._bind_cloud(new)
        return index_map, reasons

    def _alloc_pairs(self, cap):
        cap = int(cap)
        for b in self.bufs:
            b.alloc_pairs(cap)
        self.capacity = cap

    def size_pairs(self, cameras, slack=1.5):
        """Measure the pair count of a few views (host sync) and size buffers."""
        worst = 0
        b = self.bufs[0]
        for cam in cameras:
            self._preprocess(cam, b)
            worst = max(worst, int(b.tile_counts.sum().item()))
        self._alloc_pairs(max(int(worst * slack), 1024))
        return worst

    def check_overflow(self):
        return bool(self.flags_all[:, 2].any().item())

    def _status(self):
        """Read the step's status back (the one host sync of a step): raise on
        invalid surfels, and return True when the views must be re-run with
        larger pair buffers (which it allocates)."""
        flags = self.flags_all.cpu()
        if int(flags[:, 0].max()):
            raise ValueError("zero-norm quaternion")
        if int(flags[:, 1].max()):
            raise ValueError("non-finite surfel colors")
        if float(self.pack.status.item()) <= 0.0:
            return False
        need = int(flags[:, 3].max())
        if need > self.capacity:
            self._alloc_pairs(int(need * 1.25) + 1024)
        self.regrows += 1
        return True

    # -- per-view stages ----------------------------------------------------
    def _preprocess(self, cam, b):
        b.tile_counts.zero_()
        camst = _lib.make_camera(cam)
        args = (ctypes.byref(self._cl), ctypes.byref(camst), ctypes.byref(self._po), self.color_source, None,
                ctypes.byref(self._envs), _lib.ptr(b.records), _lib.ptr(b.cull), None, _lib.ptr(b.tile_counts),
                _lib.ptr(b.bininfo), ctypes.byref(b.aux) if self.color_source == _lib.SS_COLOR_IBL else None,
                _lib.ptr(b.flags))
        if self._prepared:  # inside a step: this step's prepass
            rc = self.lib.ss_preprocess_prepared(*args, _lib.ptr(self._prepass), _lib.stream_ptr())
        else:
            rc = self.lib.ss_preprocess(*args, _lib.stream_ptr())
        _lib.check(rc, "ss_preprocess")
        return camst

    def view(self, cam, target, b=None, target_done=None, mask=None):
        """Forward + backward of one view on the CURRENT stream with buffer set
        b; gradients accumulate into self.grads and b's derived-map sums.
        target_done: event recorded once `target` is consumed."""
        b = b if b is not None else self.bufs[0]
        camst = self._front(cam, b)
        self._raster(target, b, target_done=target_done, mask=mask)
        self._chain(camst, b)

    def _front(self, cam, b):
        """Stage 1 of a view (current stream): preprocess + shading, binning
        and the per-tile sort into buffer set b; returns the native camera."""
        lib = self.lib
        s = _lib.stream_ptr()
        ev = self._ev_begin("preprocess")
        camst = self._preprocess(cam, b)
        self._ev_end(ev)
        ev = self._ev_begin("bin_sort")
        _lib.check(lib.ss_bin_sort(self.n, _lib.ptr(b.bininfo), _lib.ptr(b.cull), self.W, self.H, self.tile,
                                   _lib.ptr(b.tile_counts), _lib.ptr(b.offsets), _lib.ptr(b.cursors),
                                   _lib.ptr(b.keys), _lib.ptr(b.pair), _lib.ptr(b.pair_rect), b.capacity,
                                   _lib.ptr(b.flags), _lib.ptr(b.tile_order), s),
                   "ss_bin_sort")
        self._ev_end(ev)
        return camst

    def _raster(self, target, b, target_done=None, mask=None):
        """Stage 2 (current stream): fused forward + loss + layer coefficients,
        then the record-parallel backward into b's accumulator rows."""
        lib = self.lib
        s = _lib.stream_ptr()
        ev = self._ev_begin("train_forward")
        if self.loss_mode == "l1":
            rgb_out = None
            if self.captured_rgb is not None:  # diagnostics: keep each view's fused-forward image
                rgb_out = torch.empty((self.H, self.W, 3), device=target.device, dtype=torch.float32)
                self.captured_rgb.append(rgb_out)
            _lib.check(lib.ss_train_forward(self.W, self.H, self.tile, _lib.ptr(b.offsets), _lib.ptr(b.pair),
                                            _lib.ptr(b.pair_rect), _lib.ptr(b.records), self._bg[0], self.k_max,
                                            _lib.ptr(target), _lib.ptr(b.coef), _lib.ptr(b.thr), _lib.ptr(b.pix_hdr),
                                            _lib.ptr(self.loss), _lib.ptr(rgb_out), None, _lib.ptr(b.tile_order), s),
                       "ss_train_forward")
        else:
            # deferred loss: image -> loss kernels -> layer coefficients
            cons = self.cons_scale > 0.0
            if cons:
                b.alloc_zstats(self.k_max, self.W, self.H)
                _lib.check(lib.ss_train_forward_zstats(self.W, self.H, self.tile, _lib.ptr(b.offsets),
                                                       _lib.ptr(b.pair), _lib.ptr(b.pair_rect), _lib.ptr(b.records),
                                                       self._bg[0], self.k_max, _lib.ptr(b.coef), _lib.ptr(b.thr),
                                                       _lib.ptr(b.pix_hdr), _lib.ptr(b.rgb), _lib.ptr(b.alpha),
                                                       _lib.ptr(b.tile_order), _lib.ptr(b.zst), s),
                           "ss_train_forward_zstats")
            else:
                _lib.check(lib.ss_train_forward(self.W, self.H, self.tile, _lib.ptr(b.offsets), _lib.ptr(b.pair),
                                                _lib.ptr(b.pair_rect), _lib.ptr(b.records), self._bg[0], self.k_max,
                                                None, _lib.ptr(b.coef), _lib.ptr(b.thr), _lib.ptr(b.pix_hdr), None,
                                                _lib.ptr(b.rgb), _lib.ptr(b.alpha), _lib.ptr(b.tile_order), s),
                           "ss_train_forward")
            if self.captured_rgb is not None:
                self.captured_rgb.append(b.rgb.clone())
            out = b.imgloss(b.rgb, target, b.g_rgb, self.lambda_ssim, self.tone, grad64=b.g_rgb64)
            b.loss_part += out[0:1]
            g_alpha = None
            if mask is not None and self.lambda_sil > 0.0:
                _lib.check(lib.ss_silhouette_loss(self.W * self.H, _lib.ptr(b.alpha), _lib.ptr(mask), _lib.ptr(b.sil),
                                                  _lib.ptr(b.g_alpha), _lib.ptr(b.sil_ws), s), "ss_silhouette_loss")
                b.g_alpha.mul_(self.lambda_sil)
                b.loss_part += self.lambda_sil * b.sil
                g_alpha = b.g_alpha
            if cons:
                _lib.check(lib.ss_train_coefs_cons(self.W, self.H, self.k_max, _lib.ptr(b.pix_hdr), _lib.ptr(b.coef),
                                                   _lib.ptr(b.zst), _lib.ptr(b.g_rgb), _lib.ptr(b.g_rgb64),
                                                   _lib.ptr(g_alpha), self._bg[0],
                                                   self.cons_scale, _lib.ptr(b.loss_part), s), "ss_train_coefs_cons")
            else:
                _lib.check(lib.ss_train_coefs(self.W, self.H, self.k_max, _lib.ptr(b.pix_hdr), _lib.ptr(b.coef),
                                              _lib.ptr(b.g_rgb), _lib.ptr(b.g_rgb64), _lib.ptr(g_alpha), self._bg[0],
                                              s), "ss_train_coefs")
        self._ev_end(ev)
        if target_done is not None:
            target_done.record()
        ev = self._ev_begin("train_backward")
        if self.loss_mode == "photometric" and self.cons_scale > 0.0:
            _lib.check(lib.ss_train_backward_records_cons(self.n, _lib.ptr(b.cull), _lib.ptr(b.records), self.W,
                                                          self.H, self.k_max, _lib.ptr(b.coef), _lib.ptr(b.thr),
                                                          _lib.ptr(b.pix_hdr), _lib.ptr(b.zst), _lib.ptr(b.pixel_ndc),
                                                          _lib.ptr(b.acc), _lib.ptr(b.acc64), s),
                       "ss_train_backward_records_cons")
        else:
            _lib.check(lib.ss_train_backward_records(self.n, _lib.ptr(b.cull), _lib.ptr(b.records), self.W,
                                                     self.H, self.k_max, _lib.ptr(b.coef), _lib.ptr(b.thr),
                                                     _lib.ptr(b.pix_hdr), _lib.ptr(b.pixel_ndc), _lib.ptr(b.acc),
                                                     _lib.ptr(b.acc64), s), "ss_train_backward_records")
        self._ev_end(ev)

    def _chain(self, camst, b):
        """Stage 3 (current stream): the per-surfel chain into the step's
        gradient buffer and b's derived-map sums."""
        lib = self.lib
        s = _lib.stream_ptr()
        ev = self._ev_begin("chain")
        # the chain kernels of concurrent views may overlap: their parameter
        # gradients are vector reductions (atomic), the derived-map sums go to
        # this buffer set's own float32 maps
        args = (ctypes.byref(self._cl), ctypes.byref(camst), ctypes.byref(self._po), _lib.SS_COLOR_IBL,
                ctypes.byref(self._envs), _lib.ptr(b.cull), _lib.ptr(b.acc), _lib.ptr(b.acc64),
                _lib.ptr(b.cells) if self.color_source == _lib.SS_COLOR_IBL else None, ctypes.byref(b.gs))
        if self._diffuse_per_step():
            # the diffuse taps are applied once per step (ss_diffuse_scatter at the join)
            _lib.check(lib.ss_chain_backward_prepared(*args, _lib.ptr(self._prepass), _lib.ptr(self._g_ld), s),
                       "ss_chain_backward_prepared")
        else:
            _lib.check(lib.ss_chain_backward(*args, s), "ss_chain_backward")
            # fold this view's float32 derived-map sums into the buffer set's
            # float64 ones (same stream: no ordering with the other sets)
            _lib.check(lib.ss_env_grad_merge(b.d_diff4.numel() // 4, _lib.ptr(b.d_diff4), _lib.ptr(b.d_diffuse64),
                                             s), "ss_env_grad_merge")
        _lib.check(lib.ss_env_grad_merge(b.d_spec4.numel() // 4, _lib.ptr(b.d_spec4), _lib.ptr(b.d_spec64), s),
                   "ss_env_grad_merge")
        self._ev_end(ev)

    def _diffuse_per_step(self):
        """Inside a step with the IBL prepass (float32 and float64 maps): the
        chain's diffuse lookup state comes from the prepass and its env taps are
        applied once per step (ss_diffuse_scatter at the join)."""
        e = self._envs
        return (self._prepared and self.color_source == _lib.SS_COLOR_IBL and e is not None and
                bool(e.diffuse4) and bool(e.diffuse) and bool(e.diffuse64) and bool(e.specular64))

    def _run_views(self, cameras, targets_for, target_done=None, masks=None):
        """Issue every view, alternating the worker streams (view i uses stream
        and buffers i % S); the streams are independent until the join."""
        main = torch.cuda.current_stream()
        # the view-independent per-surfel state, once for the step's views
        _lib.check(self.lib.ss_surfel_prepass(ctypes.byref(self._cl), ctypes.byref(self._envs),
                                              _lib.ptr(self._prepass), _lib.stream_ptr()), "ss_surfel_prepass")
        self._prepared = True
        diffuse_per_step = self._diffuse_per_step()
        for st in self.streams:
            st.wait_stream(main)
        nst = min(len(self.streams), self.active_streams or len(self.streams))
        try:
            for i, cam in enumerate(cameras):
                k = i % nst
                with torch.cuda.stream(self.streams[k]):
                    tgt = targets_for(i, self.streams[k])
                    self.view(cam, tgt, self.bufs[k],
                              target_done=None if target_done is None else target_done[i % len(target_done)],
                              mask=None if masks is None else masks[i])
                    if self.collect_stats:
                        b = self.bufs[k]
                        self._pairs.append(int(b.offsets[-1].item()))
                        self._kept.append(int((b.cull == 0).sum().item()))
                        self._layer_px.append(self._view_layer_pixels(b))
        finally:
            self._prepared = False
        for st in self.streams:
            main.wait_stream(st)
        if diffuse_per_step:
            _lib.check(self.lib.ss_diffuse_scatter(self.n, ctypes.byref(self._envs), _lib.ptr(self._prepass),
                                                   _lib.ptr(self._g_ld), _lib.ptr(self.d_diffuse),
                                                   _lib.stream_ptr()), "ss_diffuse_scatter")
        for b in self.bufs[1:nst]:  # the other sets' derived-map sums into the step's
            self.d_diffuse.add_(b.d_diffuse64)
            self.d_spec.add_(b.d_spec64)
            b.d_diffuse64.zero_()
            b.d_spec64.zero_()

    def _ev_begin(self, name):
        if self.kernel_events is None:
            return None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()  # on the current (worker) stream
        return (name, a, b)

    def _ev_end(self, ev):
        if ev is not None:
            ev[2].record()
            self.kernel_events.append(ev)

    @property
    def launches_per_step(self):
        return self.launches_per_view * self._nviews + self.launches_per_step_fixed

    def _view_layer_pixels(self, b):
        """Sum over pixels of the layer count of the view just run on buffer
        set b (pixels of tiles with pairs; the others hold no header)."""
        t = self.tile
        ntx, nty = self.ntx, self.ntiles // self.ntx
        live = (b.offsets[1:self.ntiles + 1] > b.offsets[:self.ntiles]).view(nty, ntx)
        live = live.repeat_interleave(t, 0).repeat_interleave(t, 1)[:self.H, :self.W].reshape(-1)
        layers = (b.pix_hdr[:, 0] >> 8) & 0xff
        return int((layers * live).sum().item())

    def last_stats(self):
        """Pair and kept-record counts and layer-pixels of the last step's
        views (collect_stats; host syncs)."""
        return {"pairs_mean": float(np.mean(self._pairs)) if self._pairs else 0.0,
                "kept_mean": float(np.mean(self._kept)) if self._kept else 0.0,
                "layer_pixels_mean": float(np.mean(self._layer_px)) if getattr(self, "_layer_px", None) else 0.0}

    @property
    def touched(self):
        """Per-surfel number of this step's views (on this rank, or summed
        over ranks after the all-reduce) in which the surfel covered a pixel."""
        return self.view_count

    def zero(self):
        self.flat.zero_()
        for b in self.bufs:
            b.d_diffuse64.zero_()
            b.d_spec64.zero_()
        self.loss.zero_()
        for b in self.bufs:
            b.loss_part.zero_()
        for b in self.bufs:
            b.flags.zero_()

    def set_normal_consistency(self, index, lambda_nc):
        """Add lambda_nc * normal_consistency_loss(cloud, index) per VIEW of
        the step (its quaternion gradient and value; train.py:216-221).  The
        reference adds the term once per single-view step; a batched step is
        the sum of its views' reference steps, so the term enters once per
        view: each rank adds lambda_nc x (its view count), and the all-reduce
        makes it lambda_nc x (views in the global step).  The index is the
        caller's NeighborIndex (rebuilt on its own schedule, like the
        reference's); pass index=None to turn the term off."""
        self._nc = None if index is None or float(lambda_nc) == 0.0 else (index, float(lambda_nc))

    def _normal_consistency(self, nviews):
        nc = getattr(self, "_nc", None)
        if nc is None or nviews == 0:
            return
        index, lam = nc
        lam = lam * nviews
        n = self.n
        if index.neighbors.shape[0] != n:
            raise ValueError("normal-consistency index built for a different cloud size")
        dev = self.cloud.centers.device
        val = torch.zeros(1, device=dev, dtype=torch.float64)
        g_n = torch.empty((n, 3), device=dev, dtype=torch.float64)
        g_q = torch.zeros((n, 4), device=dev, dtype=torch.float32)
        _lib.check(self.lib.ss_normal_consistency(n, index.neighbors.shape[1], _lib.ptr(self.cloud.centers),
                                                  _lib.ptr(self.cloud.quats), _lib.ptr(index.neighbors),
                                                  _lib.ptr(index.mean_dist), _lib.ptr(val), _lib.ptr(g_n),
                                                  _lib.ptr(g_q), _lib.stream_ptr()), "ss_normal_consistency")
        self.grads["quats"].view(-1).add_(g_q.view(-1), alpha=lam)
        self.loss.add_(val, alpha=lam)

    def gradients(self, cameras, targets, masks=None):
        """Sum of per-view gradients over this rank's views (+ env adjoint),
        all-reduced over the process group.  Re-runs the views once the pair
        buffers have grown if any rank's binning overflowed."""
        if self.capacity == 0:
            self.size_pairs(cameras[:2])
        while True:
            self.zero()
            self._nviews = len(cameras)
            self._pairs, self._kept, self._layer_px = [], [], []
            self._run_views(cameras, lambda i, st: targets[i], masks=masks)
            self._normal_consistency(len(cameras))
            self._finish()
            if not self._status():
                return

    def _env_adjoint(self):
        he, we = self.env.shape
        from .shading import env_ops
        ops = env_ops(he, we, self.env.levels, self.env.spec_samples)
        _lib.check(self.lib.ss_env_adjoint(he, we, self.env.levels, self.env.spec_samples, _lib.ptr(self.env.base64),
                                           ops.ref(), _lib.ptr(self.d_diffuse),
                                           _lib.ptr(self.d_spec), _lib.ptr(self.d_base), _lib.ptr(self.g_env_log),
                                           _lib.stream_ptr()), "ss_env_adjoint")

    def _finish(self):
        """Env adjoint + all-reduce.  The per-surfel bucket (params, ss_grad,
        view counts: 60 B/surfel) is final once the last view's chain kernel
        ran, so its all-reduce starts right then on NCCL's stream and
        overlaps the env adjoint; the small env/loss/status bucket follows
        the adjoint.  The optimiser waits for both."""
        work = self.pack.all_reduce_surfels(self.pg)
        self._env_adjoint()
        for b in self.bufs:
            self.loss += b.loss_part
        self.loss_f.copy_(self.loss)
        self.pack.status.copy_(self.flags_all[:, 2].amax())
        self.pack.all_reduce_rest(self.pg)
        if work is not None:
            work.wait()

    def fixed_costs(self):
        """CUDA-event times (ms, current stream) of the per-step fixed stages,
        each run once more on the current state (SURVEY §8d reports them beside
        the per-view numbers): env adjoint, all-reduce, Adam (+ quaternion
        renorm), env refresh.  Leaves the parameters one Adam step further."""
        def timed(fn):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            return a.elapsed_time(b)
        items = [(k, getattr(self.cloud, k), self.grads[k], self.lrs[k]) for k in PARAMS]
        items.append(("env_base_log", self.env.base_log, self.g_env_log, self.lrs["env_base_log"]))
        return {"env_adjoint": timed(self._env_adjoint),
                "allreduce": timed(lambda: self.pack.all_reduce(self.pg)),
                "adam": timed(lambda: self.adam.step_multi(items, renorm_quats="quats")),
                "env_refresh": timed(self.env.refresh)}

    def apply(self, lr_scale=1.0):
        """Adam on all tensors, quaternion renorm, env refresh (train.py:241-248)."""
        items = [(k, getattr(self.cloud, k), self.grads[k], self.lrs[k] * lr_scale) for k in PARAMS]
        items.append(("env_base_log", self.env.base_log, self.g_env_log, self.lrs["env_base_log"] * lr_scale))
        self.adam.step_multi(items, renorm_quats="quats")  # one launch, quaternions renormalised in it
        self.env.refresh(self.adam.p64.get("env_base_log"))

    # -- CUDA-graph replay ----------------------------------------------------
    MAX_GRAPHS = 8

    def _graph_key(self, cameras, targets, masks):
        cams = b"".join(bytes(_lib.make_camera(c)) for c in cameras)
        ptrs = tuple(int(t.data_ptr()) for t in targets)
        mptrs = None if masks is None else tuple(int(m.data_ptr()) for m in masks)
        return (cams, ptrs, mptrs, self.cons_scale, self.capacity, self.n, len(self.streams), self.active_streams)

    def gradients_graphed(self, cameras, targets, masks=None):
        """gradients() replayed from a CUDA graph: the first call with a given
        camera list and input tensors runs eagerly and then captures the whole
        gradient pass (every view's launches on the worker streams, the env
        adjoint, the status copy); later calls replay it with ONE host launch.
        Kernel arguments (cameras, the consolidation weight) are baked into the
        graph, so the cache is keyed by them and by the input tensors' device
        addresses; it is dropped when the pair buffers grow or the cloud is
        rebound.  The status read and the overflow re-run stay as in
        gradients().  Single process only (the NCCL all-reduce is not captured)."""
        if self.pg is not None or collectives_on():
            return self.gradients(cameras, targets, masks)
        if self.kernel_events is not None or self.collect_stats or self.captured_rgb is not None:
            return self.gradients(cameras, targets, masks)
        if self.capacity == 0:
            self.size_pairs(cameras[:2])
        key = self._graph_key(cameras, targets, masks)
        g = self._graphs.get(key)
        if g is None:
            self.gradients(cameras, targets, masks)  # eager: sizes buffers, sets kernel attributes
            key = self._graph_key(cameras, targets, masks)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.zero()
                self._nviews = len(cameras)
                self._run_views(cameras, lambda i, st: targets[i], masks=masks)
                self._normal_consistency(len(cameras))
                self._finish()
            if len(self._graphs) >= self.MAX_GRAPHS:
                self._graphs.pop(next(iter(self._graphs)))
            self._graphs[key] = g
            return  # the eager pass's gradients stand (capture runs nothing)
        g.replay()
        if self._status():  # pair buffers grew: the captured launches are stale
            self._graphs.clear()
            self.gradients(cameras, targets, masks)

    def step(self, cameras, targets, masks=None, graph=False):
        """One optimisation step over `cameras` (gradients, Adam, env refresh);
        graph=True replays the gradient pass from a CUDA graph (see
        gradients_graphed)."""
        if graph:
            self.gradients_graphed(cameras, targets, masks)
        else:
            self.gradients(cameras, targets, masks)
        self.apply()
        # device scalar: loss="l1": sum over views of sum|rgb - target|;
        # loss="photometric": sum over views of the per-view fit loss
        return self.loss_f

    def step_host(self, cameras, host_targets):
        """step() with the targets in pinned HOST memory: each view's target is
        copied on a side stream into a ring of staging buffers (one more than
        the worker streams, so a copy never waits on a view still in flight on
        another stream), overlapped with the previous views' kernels."""
        if self.capacity == 0:
            self.size_pairs(cameras[:2])
        nst = len(self.streams) + 1
        if self._stage is None or len(self._stage) != nst:
            self._stage = [torch.empty((self.H, self.W, 3), device=self.pack.flat.device, dtype=torch.float32)
                           for _ in range(nst)]
            self._copy = torch.cuda.Stream()
        ready = [torch.cuda.Event() for _ in range(nst)]
        free = [torch.cuda.Event() for _ in range(nst)]
        main = torch.cuda.current_stream()
        self._copy.wait_stream(main)

        def issue(i):
            k = i % nst
            with torch.cuda.stream(self._copy):
                if i >= nst:
                    self._copy.wait_event(free[k])
                self._stage[k].copy_(host_targets[i], non_blocking=True)
                ready[k].record(self._copy)

        def target_for(i, stream):
            # view i's target is copied while the previous views compute
            if i + 1 < len(cameras):
                issue(i + 1)
            stream.wait_event(ready[i % nst])
            return self._stage[i % nst]

        while True:
            self.zero()
            self._nviews = len(cameras)
            issue(0)
            self._run_views(cameras, target_for, target_done=free)
            self._normal_consistency(len(cameras))
            self._finish()
            if not self._status():
                break
        self.apply()
        return self.loss_f
