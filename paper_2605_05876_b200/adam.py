"""Adam over named device tensors (mirror of surfsplat.adam, adam.py:12-81).

Each step is one fused native kernel (csrc/optim.cu) per parameter tensor:
moments and the parameter are read and written once.  State is float32 on
the device (the reference keeps float64 numpy moments); the update itself is
evaluated in float64 per element.
"""

from __future__ import annotations

import torch

from . import _lib


class Adam:
    def __init__(self, beta1=0.9, beta2=0.999, eps=1e-15):
        self.beta1, self.beta2, self.eps = float(beta1), float(beta2), float(eps)
        self.m: dict[str, torch.Tensor] = {}
        self.v: dict[str, torch.Tensor] = {}
        self.t: dict[str, int] = {}

    def step(self, name, param, grad, lr):
        if tuple(grad.shape) != tuple(param.shape):
            raise ValueError(f"gradient shape {tuple(grad.shape)} != param shape {tuple(param.shape)}")
        if name not in self.m:
            self.m[name] = torch.zeros_like(param, dtype=torch.float32)
            self.v[name] = torch.zeros_like(param, dtype=torch.float32)
            self.t[name] = 0
        self.t[name] += 1
        g = grad.to(torch.float32).contiguous()
        lib = _lib.load()
        rc = lib.ss_adam_step(param.numel(), _lib.ptr(param), _lib.ptr(g), _lib.ptr(self.m[name]),
                              _lib.ptr(self.v[name]), self.t[name], float(lr), self.beta1, self.beta2, self.eps,
                              _lib.stream_ptr())
        _lib.check(rc, "ss_adam_step")
        return param

    def remap(self, name, index):
        """adam.py:43-58: reindex rows; index -1 rows start from zero."""
        if name not in self.m:
            return
        idx = torch.as_tensor(index, device=self.m[name].device, dtype=torch.int64)
        keep = idx >= 0
        src = torch.where(keep, idx, torch.zeros_like(idx))
        for store in (self.m, self.v):
            new = store[name][src].clone()
            new[~keep] = 0.0
            store[name] = new.contiguous()

    def remap_all(self, index):
        for name in list(self.m):
            self.remap(name, index)

    def state_arrays(self):
        out = {}
        for name in self.m:
            out[f"adam_m_{name}"] = self.m[name].cpu().numpy()
            out[f"adam_v_{name}"] = self.v[name].cpu().numpy()
            out[f"adam_t_{name}"] = self.t[name]
        return out


def normalize_quats(quats):
    lib = _lib.load()
    _lib.check(lib.ss_normalize_quats(quats.shape[0], _lib.ptr(quats), _lib.stream_ptr()), "ss_normalize_quats")
    return quats
