"""CUDA image losses (csrc/losses.cu) against the reference's golden outputs
and the oracle restatement (needs a B200)."""

import os

import numpy as np
import pytest
import torch

from parity import host
from oracle import oracle as O

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "losses.npz")


def _close(got, ref, rel=1e-6, floor=1e-7):
    """float32 outputs of float64 math: relative bound + array-scaled floor."""
    a = host(got).astype(np.float64)
    b = np.asarray(ref, dtype=np.float64)
    scale = max(float(np.abs(b).max()), 1e-30)
    err = np.abs(a - b)
    bad = err > rel * np.maximum(np.abs(a), np.abs(b)) + floor * scale
    return int(bad.sum()), float(err.max() / scale)


def test_losses_match_reference_goldens():
    d = np.load(GOLD)
    x, y, g_up = d["img"], d["tgt"], d["g_up"]
    for mode in ("ldr", "hdr-loss"):
        k = mode.replace("-", "_")
        assert _close(ss.tone_map(x, mode), d["tone_" + k])[0] == 0
        assert _close(ss.tone_map_backward(x, mode, g_up.astype(np.float32)),
                      O.tone_map_backward(x, mode, g_up.astype(np.float32)))[0] == 0
        for lam in (0.0, 0.2):
            v, g = ss.image_loss(x, y, tone=mode, lambda_ssim=lam)
            # reference: photometric_loss on the tone-mapped images, chained through tone_map_backward
            ref_v = float(d[f"photo_{k}_{int(lam * 10)}"])
            ref_g = O.tone_map_backward(x, mode, d[f"photo_grad_{k}_{int(lam * 10)}"])
            assert v == pytest.approx(ref_v, rel=1e-12)
            assert _close(g, ref_g)[0] == 0, (mode, lam, _close(g, ref_g))
    v, g = ss.ssim_loss(x, y)
    assert v == pytest.approx(float(d["ssim"]), rel=1e-12)
    assert _close(g, d["ssim_grad"])[0] == 0
    v, g = ss.ssim_loss(d["alpha"], d["mask"])
    assert v == pytest.approx(float(d["ssim_1c"]), rel=1e-12)
    assert _close(g, d["ssim_1c_grad"])[0] == 0
    v, g = ss.silhouette_loss(d["alpha"], d["mask"])
    assert v == pytest.approx(float(d["sil"]), rel=1e-12)
    assert _close(g, d["sil_grad"])[0] == 0


@pytest.mark.parametrize("shape", [(800, 800, 3), (37, 53, 3), (11, 11, 1), (9, 30, 3)])
def test_photometric_loss_matches_oracle(shape):
    """Full-size and ragged images (tile edges, the window-sized minimum, and
    an image smaller than the window where SSIM is defined as 0)."""
    rng = np.random.default_rng(3)
    x = np.exp(rng.normal(-1.0, 1.0, shape)).astype(np.float32)
    y = np.exp(rng.normal(-1.0, 1.0, shape)).astype(np.float32)
    if shape[2] == 1:
        x, y = x[..., 0], y[..., 0]
    v, g = ss.image_loss(x, y, tone="hdr-loss", lambda_ssim=0.2)
    mx, my = O.tone_map(x, "hdr-loss"), O.tone_map(y, "hdr-loss")
    rv, rg = O.photometric_loss(mx, my, 0.2)
    rg = O.tone_map_backward(x, "hdr-loss", rg)
    assert v == pytest.approx(rv, rel=1e-11)
    bad, err = _close(g, rg)
    assert bad == 0, err


def test_loss_errors_like_reference():
    with pytest.raises(ValueError):
        ss.photometric_loss(np.zeros((4, 4, 3), np.float32), np.zeros((4, 5, 3), np.float32))
    with pytest.raises(ValueError):
        ss.tone_map(np.zeros(3, np.float32), "srgb")
    with pytest.raises(ValueError):
        ss.silhouette_loss(np.zeros((4, 4), np.float32), np.zeros((4, 3), np.float32))
    # empty union: zero loss and gradient (losses.py:120-121)
    v, g = ss.silhouette_loss(np.zeros((6, 6), np.float32), np.zeros((6, 6), np.float32))
    assert v == 0.0 and float(torch.abs(g).max()) == 0.0
