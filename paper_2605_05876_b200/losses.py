"""Image losses used at the render/backward boundary (losses.py:94-123).

photometric_loss with lambda_ssim = 0 (the BASELINE config-0 L1) and
silhouette_loss on device tensors.  The SSIM variant is SURVEY §8(f) row 1
(next round); asking for it raises instead of silently falling back.
"""

from __future__ import annotations

import torch


def photometric_loss(img, target, lambda_ssim=0.2):
    x = torch.as_tensor(img)
    y = torch.as_tensor(target, device=x.device, dtype=x.dtype)
    if x.shape != y.shape:
        raise ValueError("image shape mismatch")
    if lambda_ssim != 0.0:
        raise NotImplementedError("SSIM term: SURVEY §8(f) row 1, not yet on the B200 path")
    diff = x - y
    return float(diff.abs().mean().item()), torch.sign(diff) / diff.numel()


def silhouette_loss(alpha, mask):
    a = torch.as_tensor(alpha)
    m = torch.as_tensor(mask, device=a.device, dtype=a.dtype)
    if a.shape != m.shape:
        raise ValueError("image shape mismatch")
    inter = float((a * m).sum().item())
    union = float((a + m - a * m).sum().item())
    if union <= 0.0:
        return 0.0, torch.zeros_like(a)
    return 1.0 - inter / union, (inter * (1.0 - m) - m * union) / (union * union)
