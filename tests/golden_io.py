"""Load the golden fixtures (tests/golden/*.npz, made by make_golden.py from
the reference implementation) into plain objects."""

from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENES = ("explicit_cons", "albedo_nomip", "ibl_env", "kmax_stack", "culling", "config0_small")
CLOUD_KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw")


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as f:
        return {k: f[k] for k in f.files}


def cloud_of(d, prefix="cloud_"):
    return SimpleNamespace(**{k: d[prefix + k] for k in CLOUD_KEYS})


def camera_of(d):
    w, h = (int(x) for x in d["cam_wh"])
    return SimpleNamespace(view=d["cam_view"], proj=d["cam_proj"], width=w, height=h)


def proj_of(d):
    """Reference ProjectedSurfels (kept rows) as an oracle-style dict."""
    p = {k[len("proj_"):]: d[k] for k in d if k.startswith("proj_")}
    p["z_start"] = (p["view_z"] - p["eps_z"]).astype(np.float32)
    p["z_end"] = (p["view_z"] + p["eps_z"]).astype(np.float32)
    w, h = (int(x) for x in d["cam_wh"])
    p["width"], p["height"] = w, h
    p["mip_enabled"] = bool(d["mip_enabled"])
    p["mip_sigma"] = 0.1
    return p
