"""Tolerance helpers shared by the GPU parity tests (north_star: images and
depth within 1e-4 relative, parameter gradients within 1e-3 relative)."""

import numpy as np
import torch


def host(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def image_close(got, ref, rel=1e-4, abs_=1e-6):
    """|a-b| <= rel*max(|a|,|b|) + abs  (SURVEY §8c image tolerance)."""
    a = host(got).astype(np.float64)
    b = host(ref).astype(np.float64)
    bad = np.abs(a - b) > rel * np.maximum(np.abs(a), np.abs(b)) + abs_
    return int(bad.sum()), float(np.max(np.abs(a - b))) if a.size else 0.0


def grad_close(got, ref, rel=1e-3, floor=1e-5):
    """|a-b| <= rel*max(|a|,|b|) + floor*max|ref|: the relative bound with an
    array-scaled absolute floor (gradcheck.py:180 uses an absolute 1e-6)."""
    a = host(got).astype(np.float64)
    b = host(ref).astype(np.float64)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-30)
    err = np.abs(a - b)
    bad = err > rel * np.maximum(np.abs(a), np.abs(b)) + floor * scale
    return int(bad.sum()), float(err.max() / scale) if a.size else 0.0


def grad_outliers(got, ref, rel=1e-3, floor=1e-5, top=8):
    """The entries grad_close rejects, worst first: (flat index, got, ref,
    |a-b| / max|ref|, |a-b| / max(|a|,|b|)) -- printed by the full-size tests
    so every out-of-tolerance entry is visible with its magnitude."""
    a = host(got).astype(np.float64).reshape(-1)
    b = host(ref).astype(np.float64).reshape(-1)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-30)
    err = np.abs(a - b)
    bad = np.flatnonzero(err > rel * np.maximum(np.abs(a), np.abs(b)) + floor * scale)
    order = bad[np.argsort(-err[bad])][:top]
    return [(int(i), float(a[i]), float(b[i]), float(err[i] / scale),
             float(err[i] / max(abs(a[i]), abs(b[i]), 1e-300))) for i in order], int(bad.size)
