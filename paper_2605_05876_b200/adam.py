"""Adam over named device tensors (mirror of surfsplat.adam, adam.py:12-81).

Each step is one fused native kernel (csrc/optim.cu) per parameter tensor
(or one launch for all of them, step_multi): moments and the parameter are
read and written once.  The moments are float64 by default, like the
reference's numpy state (adam.py:26-28), so checkpoints carry the same
dtypes; state_dtype=torch.float32 halves their memory and traffic.  The
update itself is evaluated in float64 per element either way.

master_params=True keeps a float64 master copy of every parameter it steps
(`p64`), like the reference's fit, which promotes the cloud to float64
(train.py:168-174): step_multi then runs the reference's numpy update
operation by operation on the masters (ss_adam_multi_master, float64
hyper-parameters) and writes the float32 rounding into the tensors the
kernels read.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


class Adam:
    def __init__(self, beta1=0.9, beta2=0.999, eps=1e-15, state_dtype=torch.float64, master_params=False):
        if state_dtype not in (torch.float64, torch.float32):
            raise ValueError("state_dtype must be torch.float64 or torch.float32")
        if master_params and state_dtype != torch.float64:
            raise ValueError("master parameters need float64 moments")
        self.beta1, self.beta2, self.eps = float(beta1), float(beta2), float(eps)
        self.state_dtype = state_dtype
        self.master_params = bool(master_params)
        self.m: dict[str, torch.Tensor] = {}
        self.v: dict[str, torch.Tensor] = {}
        self.t: dict[str, int] = {}
        self.p64: dict[str, torch.Tensor] = {}  # float64 masters (master_params)

    def step(self, name, param, grad, lr):
        if self.master_params:
            return self.step_multi([(name, param, grad, lr)])[0]
        if tuple(grad.shape) != tuple(param.shape):
            raise ValueError(f"gradient shape {tuple(grad.shape)} != param shape {tuple(param.shape)}")
        self._init_state(name, param)
        self.t[name] += 1
        g = grad.to(torch.float32).contiguous()
        lib = _lib.load()
        fn = lib.ss_adam_step_f64 if self.state_dtype == torch.float64 else lib.ss_adam_step
        rc = fn(param.numel(), _lib.ptr(param), _lib.ptr(g), _lib.ptr(self.m[name]), _lib.ptr(self.v[name]),
                self.t[name], float(lr), self.beta1, self.beta2, self.eps, _lib.stream_ptr())
        _lib.check(rc, "ss_adam_step")
        return param

    def _init_state(self, name, param):
        if name not in self.m:
            self.m[name] = torch.zeros_like(param, dtype=self.state_dtype)
            self.v[name] = torch.zeros_like(param, dtype=self.state_dtype)
            self.t[name] = 0
        elif self.m[name].dtype != self.state_dtype:
            raise ValueError(f"optimizer state {name!r} is {self.m[name].dtype}, not {self.state_dtype}")
        if self.master_params:
            p = self.p64.get(name)
            if p is None or p.shape != param.shape:  # first use, or the tensor was replaced
                self.p64[name] = param.detach().to(torch.float64).contiguous()

    def set_master(self, name, values):
        """Replace the float64 master of `name` (e.g. a loaded float64
        checkpoint); the float32 tensor the kernels read is the caller's."""
        self.p64[name] = torch.as_tensor(values, device="cuda", dtype=torch.float64).contiguous()

    def step_multi(self, items, renorm_quats=None):
        """Adam on several tensors in ONE fused launch (csrc/optim.cu
        ss_adam_multi): items = [(name, param, grad, lr), ...]; the tensor
        named `renorm_quats` (n, 4) is renormalised right after its update
        (train.py:241-246).  Same arithmetic as step() per tensor."""
        import ctypes
        if not 1 <= len(items) <= 8:
            raise ValueError("step_multi takes 1..8 tensors")
        cols = {k: [] for k in ("p", "g", "m", "v", "n", "t", "lr", "q")}
        keep = []
        for name, param, grad, lr in items:
            if tuple(grad.shape) != tuple(param.shape):
                raise ValueError(f"gradient shape {tuple(grad.shape)} != param shape {tuple(param.shape)}")
            self._init_state(name, param)
            self.t[name] += 1
            g = grad.to(torch.float32).contiguous()
            keep.append(g)
            for key, val in (("p", param.data_ptr()), ("g", g.data_ptr()), ("m", self.m[name].data_ptr()),
                             ("v", self.v[name].data_ptr()), ("n", param.numel()), ("t", self.t[name]),
                             ("lr", float(lr)), ("q", int(name == renorm_quats))):
                cols[key].append(val)
        k = len(items)
        ptrs = {c: (ctypes.c_void_p * k)(*cols[c]) for c in ("p", "g", "m", "v")}
        lib = _lib.load()
        if self.master_params:
            masters = (ctypes.c_void_p * k)(*[self.p64[it[0]].data_ptr() for it in items])
            # bias corrections exactly as the reference's Python (1.0 - beta ** t)
            c1 = (ctypes.c_double * k)(*[1.0 - self.beta1 ** t for t in cols["t"]])
            c2 = (ctypes.c_double * k)(*[1.0 - self.beta2 ** t for t in cols["t"]])
            rc = lib.ss_adam_multi_master(k, ptrs["p"], masters, ptrs["g"], ptrs["m"], ptrs["v"],
                                          (ctypes.c_int64 * k)(*cols["n"]), c1, c2, (ctypes.c_double * k)(*cols["lr"]),
                                          (ctypes.c_int * k)(*cols["q"]), self.beta1, self.beta2, self.eps,
                                          _lib.stream_ptr())
            _lib.check(rc, "ss_adam_multi_master")
            return [it[1] for it in items]
        fn = lib.ss_adam_multi_f64 if self.state_dtype == torch.float64 else lib.ss_adam_multi
        rc = fn(k, ptrs["p"], ptrs["g"], ptrs["m"], ptrs["v"], (ctypes.c_int64 * k)(*cols["n"]),
                (ctypes.c_int * k)(*cols["t"]), (ctypes.c_float * k)(*cols["lr"]), (ctypes.c_int * k)(*cols["q"]),
                self.beta1, self.beta2, self.eps, _lib.stream_ptr())
        _lib.check(rc, "ss_adam_multi")
        return [it[1] for it in items]

    def remap(self, name, index, param=None):
        """adam.py:43-58: reindex rows; index -1 rows start from zero.  A float64
        master (master_params) is reindexed too, its new rows taken from
        `param` (the float32 tensor after the topology change); without
        `param` the master is re-seeded from the tensor at the next step."""
        if name not in self.m:
            return
        idx = torch.as_tensor(index, device=self.m[name].device, dtype=torch.int64)
        keep = idx >= 0
        src = torch.where(keep, idx, torch.zeros_like(idx))
        for store in (self.m, self.v):
            new = store[name][src].clone()
            new[~keep] = 0.0
            store[name] = new.contiguous()
        if name in self.p64:
            if param is None:
                del self.p64[name]
            else:
                new = self.p64[name][src].clone()
                new[~keep] = param[~keep].to(torch.float64)
                self.p64[name] = new.contiguous()

    def remap_all(self, index, params=None):
        for name in list(self.m):
            self.remap(name, index, None if params is None else params.get(name))

    def state_arrays(self):
        out = {}
        for name in self.m:
            out[f"adam_m_{name}"] = self.m[name].cpu().numpy()
            out[f"adam_v_{name}"] = self.v[name].cpu().numpy()
            out[f"adam_t_{name}"] = np.asarray(self.t[name], dtype=np.int64)
        return out


def _load_state(self, arrays):
    """adam.py:69-81: restore moments and step counts from checkpoint arrays."""
    self.m.clear(); self.v.clear(); self.t.clear()
    for key, val in arrays.items():
        for pre, store in (("adam_m_", self.m), ("adam_v_", self.v)):
            if key.startswith(pre):
                store[key[len(pre):]] = torch.as_tensor(np.asarray(val), device="cuda",
                                                        dtype=self.state_dtype).contiguous()
        if key.startswith("adam_t_"):
            self.t[key[len("adam_t_"):]] = int(val)
    if set(self.m) != set(self.v) or set(self.m) != set(self.t):
        raise ValueError("incomplete optimizer state")


Adam.load_state_arrays = _load_state


def normalize_quats(quats):
    lib = _lib.load()
    _lib.check(lib.ss_normalize_quats(quats.shape[0], _lib.ptr(quats), _lib.stream_ptr()), "ss_normalize_quats")
    return quats
