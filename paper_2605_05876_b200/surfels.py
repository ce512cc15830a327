"""Surfel parameters on the device (mirror of surfsplat.surfels, surfels.py:80-209).

A SurfelCloud holds six float32 CUDA tensors in struct-of-arrays layout:
centers (N,3), quats (N,4) wxyz, log_scales (N,2), albedo_raw (N,3),
metallic_raw (N,), roughness_raw (N,) -- 56 bytes per surfel, the layout the
kernels stream.  Construction accepts numpy arrays or tensors and moves them
to the current CUDA device.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np
import torch

FIELDS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw")
_SHAPES = {"centers": (3,), "quats": (4,), "log_scales": (2,), "albedo_raw": (3,),
           "metallic_raw": (), "roughness_raw": ()}


def _dev(x, device):
    if isinstance(x, torch.Tensor):
        t = x.detach()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.float32))
    return t.to(device=device, dtype=torch.float32).contiguous()


@dataclass
class SurfelCloud:
    centers: torch.Tensor
    quats: torch.Tensor
    log_scales: torch.Tensor
    albedo_raw: torch.Tensor
    metallic_raw: torch.Tensor
    roughness_raw: torch.Tensor

    def __post_init__(self):
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if device is None:
            raise RuntimeError("SurfelCloud lives on a CUDA device; none is available")
        n = None
        for name in FIELDS:
            t = _dev(getattr(self, name), device)
            want = _SHAPES[name]
            if n is None:
                n = t.shape[0]
            if t.shape[0] != n:
                raise ValueError(f"{name} has {t.shape[0]} rows, expected {n}")
            if tuple(t.shape[1:]) != want:
                raise ValueError(f"{name} must be (N{', ' + str(want[0]) if want else ''})")
            setattr(self, name, t)

    def __len__(self):
        return self.centers.shape[0]

    @classmethod
    def from_host(cls, cloud):
        """Any object with the reference's six fields (e.g. surfsplat.SurfelCloud)."""
        return cls(*(getattr(cloud, k) for k in FIELDS))

    def to_host(self):
        return {k: getattr(self, k).cpu().numpy() for k in FIELDS}

    def copy(self):
        return SurfelCloud(*(getattr(self, k).clone() for k in FIELDS))

    def select(self, index):
        return SurfelCloud(*(getattr(self, k)[index] for k in FIELDS))

    @staticmethod
    def concatenate(clouds):
        return SurfelCloud(*(torch.cat([getattr(c, k) for c in clouds]) for k in FIELDS))

    @property
    def scales(self):
        return torch.exp(self.log_scales)

    @property
    def albedo(self):
        return torch.sigmoid(self.albedo_raw)

    @property
    def metallic(self):
        return torch.sigmoid(self.metallic_raw)

    @property
    def roughness(self):
        return torch.sigmoid(self.roughness_raw)

    def params(self):
        return {k: getattr(self, k) for k in FIELDS}


def quats_from_normals(normals):
    """Unit wxyz quaternions whose frame normal (third column) is `normals`:
    shortest-arc rotation from +z, (pi about x) for normals along -z
    (same convention as surfels.py:192-209).  numpy float64, host side."""
    n = np.asarray(normals, dtype=np.float64)
    n = n / np.linalg.norm(n, axis=-1, keepdims=True)
    q = np.zeros((len(n), 4))
    q[:, 0] = 1.0 + n[:, 2]
    q[:, 1] = -n[:, 1]
    q[:, 2] = n[:, 0]
    flip = q[:, 0] < 1e-8
    q[flip] = (0.0, 1.0, 0.0, 0.0)
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def logit(y):
    y = np.asarray(y, dtype=np.float64)
    return np.log(y) - np.log1p(-y)
