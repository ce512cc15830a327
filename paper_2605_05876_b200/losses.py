"""Image losses at the render/backward boundary (losses.py:45-123), on the
CUDA kernels of csrc/losses.cu.

Same names, arguments and return convention as the reference: each returns
(value, gradient w.r.t. the first argument); values are Python floats (one
device->host read), gradients float32 CUDA tensors.  ``image_loss`` is the
fused form the training step uses: tone map -> (1 - l) L1 + l (1 - SSIM) ->
tone-map backward, with the scalar results left on the device.
"""

from __future__ import annotations

import torch

from . import _lib
from .shading import TONE_MODES

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5


def _pair(img, target):
    x = torch.as_tensor(img, device="cuda", dtype=torch.float32).contiguous()
    y = torch.as_tensor(target, device="cuda", dtype=torch.float32).contiguous()
    if x.shape != y.shape:
        raise ValueError("image shape mismatch")
    if x.dim() not in (2, 3) or (x.dim() == 3 and x.shape[2] not in (1, 3)):
        raise ValueError("images must be (H, W) or (H, W, C) with C in {1, 3}")
    return x, y


class ImageLoss:
    """Device workspace + launcher for ss_photometric_loss on (H, W, C)."""

    def __init__(self, height, width, channels=3, device="cuda"):
        self.lib = _lib.load()
        self.shape = (int(height), int(width), int(channels))
        nbytes = self.lib.ss_photometric_workspace(*self.shape)
        self.ws = torch.empty((nbytes + 7) // 8, device=device, dtype=torch.float64)
        self.out = torch.zeros(3, device=device, dtype=torch.float64)  # loss, L1, 1 - SSIM

    def __call__(self, x, y, grad, lambda_ssim=0.2, tone=None, grad64=None):
        """Launch on the current stream; returns the device `out` tensor.
        grad64 (optional): the gradient in float64 as well."""
        mode = -1 if tone is None else TONE_MODES[tone]
        if not 0.0 <= lambda_ssim <= 1.0:
            raise ValueError("lambda_ssim must lie in [0, 1]")
        h, w, c = self.shape
        _lib.check(self.lib.ss_photometric_loss(h, w, c, _lib.ptr(x), _lib.ptr(y), mode, float(lambda_ssim),
                                                _lib.ptr(self.out), _lib.ptr(grad), _lib.ptr(grad64),
                                                _lib.ptr(self.ws), _lib.stream_ptr()), "ss_photometric_loss")
        return self.out


def _run(img, target, lambda_ssim, tone=None):
    x, y = _pair(img, target)
    h, w = x.shape[:2]
    c = x.shape[2] if x.dim() == 3 else 1
    grad = torch.empty_like(x)
    out = ImageLoss(h, w, c)(x, y, grad, lambda_ssim, tone)
    return out, grad


def ssim_loss(img, target, window=SSIM_WINDOW, sigma=SSIM_SIGMA):
    """losses.py:45-91: 1 - mean SSIM over the fully windowed interior."""
    if window != SSIM_WINDOW or sigma != SSIM_SIGMA:
        raise ValueError("the B200 path implements the reference's 11x11, sigma 1.5 window only")
    out, grad = _run(img, target, 1.0)
    return float(out[2].item()), grad


def photometric_loss(img, target, lambda_ssim=0.2):
    """losses.py:94-108: (1 - lambda) L1 + lambda (1 - SSIM), gradient w.r.t. img."""
    out, grad = _run(img, target, float(lambda_ssim))
    return float(out[0].item()), grad


def image_loss(rgb, target, tone="hdr-loss", lambda_ssim=0.2):
    """train.py:194-199 fused: photometric loss of the tone-mapped images and
    its gradient w.r.t. the linear rgb (one pass, float64 inside)."""
    out, grad = _run(rgb, target, float(lambda_ssim), tone)
    return float(out[0].item()), grad


def silhouette_loss(alpha, mask):
    """losses.py:111-123: 1 - soft IoU, gradient w.r.t. alpha."""
    a, m = _pair(alpha, mask)
    lib = _lib.load()
    grad = torch.empty_like(a)
    out = torch.zeros(1, device=a.device, dtype=torch.float64)
    ws = torch.empty(2, device=a.device, dtype=torch.float64)
    _lib.check(lib.ss_silhouette_loss(a.numel(), _lib.ptr(a), _lib.ptr(m), _lib.ptr(out), _lib.ptr(grad),
                                      _lib.ptr(ws), _lib.stream_ptr()), "ss_silhouette_loss")
    return float(out.item()), grad


def normal_consistency_loss(cloud, index):
    """losses.py:189-220: mean over surfels and neighbour slots of
    w_ij (1 - n_i . n_j), w_ij = exp(-|c_i - c_j|^2 / (2 sigma_i^2)); returns
    (loss, quaternion gradient (N, 4) float32)."""
    n = len(cloud)
    if index.neighbors.shape[0] != n:
        raise ValueError("index built for a different cloud size")
    dev = cloud.centers.device
    g_q = torch.zeros((n, 4), device=dev, dtype=torch.float32)
    if n == 0:
        return 0.0, g_q
    lib = _lib.load()
    loss = torch.zeros(1, device=dev, dtype=torch.float64)
    g_n = torch.empty((n, 3), device=dev, dtype=torch.float64)
    _lib.check(lib.ss_normal_consistency(n, index.neighbors.shape[1], _lib.ptr(cloud.centers), _lib.ptr(cloud.quats),
                                         _lib.ptr(index.neighbors), _lib.ptr(index.mean_dist), _lib.ptr(loss),
                                         _lib.ptr(g_n), _lib.ptr(g_q), _lib.stream_ptr()), "ss_normal_consistency")
    return float(loss.item()), g_q
