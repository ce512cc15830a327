"""Seeded synthetic workloads for the BASELINE.json configs (host numpy).

BASELINE names no public dataset; these generators stand in with the stated
shapes, sizes and value distributions.  Geometry is
area-uniform on the named surface, radially displaced by seeded value noise;
normals are the displaced surface's (radial direction tilted by the
displacement gradient); attributes are stored raw (logit) like
SurfelCloud.from_oriented_points.
"""

from __future__ import annotations

import numpy as np

from .surfels import logit, quats_from_normals


def _value_noise(p, seed, octaves=3, base_freq=2.0):
    """Smooth 3-D value noise in [-1, 1] (trilinear with smoothstep), fBm."""
    rng = np.random.default_rng(seed)
    lat = rng.uniform(-1.0, 1.0, size=(64, 64, 64))
    out = np.zeros(len(p))
    amp, freq, norm = 1.0, base_freq, 0.0
    for _ in range(octaves):
        q = p * freq + 17.0
        i0 = np.floor(q).astype(np.int64)
        f = q - i0
        f = f * f * (3.0 - 2.0 * f)
        acc = np.zeros(len(p))
        for dx in (0, 1):
            wx = f[:, 0] if dx else 1.0 - f[:, 0]
            for dy in (0, 1):
                wy = f[:, 1] if dy else 1.0 - f[:, 1]
                for dz in (0, 1):
                    wz = f[:, 2] if dz else 1.0 - f[:, 2]
                    v = lat[(i0[:, 0] + dx) % 64, (i0[:, 1] + dy) % 64, (i0[:, 2] + dz) % 64]
                    acc += wx * wy * wz * v
        out += amp * acc
        norm += amp
        amp *= 0.5
        freq *= 2.0
    return out / norm


def _displaced_sphere(n, rng, radius, amp, octaves, seed):
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    h = _value_noise(d, seed, octaves)
    pts = d * (radius + amp * h)[:, None]
    # normal of r(d) = radius + amp*h(d): radial minus the tangential gradient
    eps = 1e-3
    grad = np.zeros((n, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = eps
        grad[:, k] = (_value_noise(d + e, seed, octaves) - _value_noise(d - e, seed, octaves)) / (2 * eps)
    tang = grad - np.sum(grad * d, axis=1, keepdims=True) * d
    nrm = d - amp * tang / (radius + amp * h)[:, None]
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return pts, nrm


def morton_order(points, bits=10):
    """Permutation sorting points along a 3-D Morton (Z-order) curve (a
    spatially coherent surfel order, e.g. for TrainStep reordering studies).
    The generators keep area-uniform sampling order: measured on B200, the
    binning counters see less contention when consecutive surfels are spread
    over the image."""
    p = np.asarray(points, dtype=np.float64)
    lo, hi = p.min(axis=0), p.max(axis=0)
    q = ((p - lo) / np.maximum(hi - lo, 1e-12) * ((1 << bits) - 1)).astype(np.uint64)

    def spread(v):
        v = v & np.uint64(0x3FF)
        v = (v | (v << np.uint64(16))) & np.uint64(0x030000FF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x0300F00F)
        v = (v | (v << np.uint64(4))) & np.uint64(0x030C30C3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x09249249)
        return v

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable")


def _raw_cloud(centers, normals, log_scales, albedo, rough, metal):
    cl = lambda x: logit(np.clip(x, 1e-5, 1 - 1e-5))
    return {
        "centers": centers.astype(np.float32),
        "quats": quats_from_normals(normals).astype(np.float32),
        "log_scales": log_scales.astype(np.float32),
        "albedo_raw": cl(albedo).astype(np.float32),
        "metallic_raw": cl(metal).astype(np.float32),
        "roughness_raw": cl(rough).astype(np.float32),
    }


def config0(seed=0, n=10_000):
    """10k surfels uniform on the unit sphere, radial normals (BASELINE cfg 0)."""
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(n, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    ls = rng.uniform(np.log(0.01), np.log(0.03), size=(n, 2))
    return _raw_cloud(p, p, ls, rng.uniform(0, 1, (n, 3)), rng.uniform(0.1, 0.9, n), rng.uniform(0, 1, n))


def config1(seed=0, n=200_000, amp=0.05, octaves=3):
    """200k surfels area-uniform on torus(R=1, r=0.35) U sphere(0.6), displaced
    along the analytic normal by 3-octave value noise (BASELINE cfg 1)."""
    rng = np.random.default_rng(seed)
    R, r, rs = 1.0, 0.35, 0.6
    a_t, a_s = 4.0 * np.pi ** 2 * R * r, 4.0 * np.pi * rs ** 2
    nt = int(round(n * a_t / (a_t + a_s)))
    # torus: area element (R + r cos v) du dv, rejection on v
    vs = np.empty(0)
    while len(vs) < nt:
        v = rng.uniform(0, 2 * np.pi, 2 * nt)
        keep = rng.uniform(0, R + r, 2 * nt) < R + r * np.cos(v)
        vs = np.concatenate([vs, v[keep]])
    v = vs[:nt]
    u = rng.uniform(0, 2 * np.pi, nt)
    nrm_t = np.stack([np.cos(v) * np.cos(u), np.cos(v) * np.sin(u), np.sin(v)], 1)
    pts_t = np.stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u), r * np.sin(v)], 1)
    d = rng.normal(size=(n - nt, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pts = np.concatenate([pts_t, rs * d])
    nrm = np.concatenate([nrm_t, d])
    pts = pts + (amp * _value_noise(pts, seed + 1, octaves))[:, None] * nrm
    ls = rng.uniform(np.log(0.005), np.log(0.02), size=(n, 2))
    return _raw_cloud(pts, nrm, ls, rng.uniform(0, 1, (n, 3)), rng.uniform(0.1, 0.9, n), rng.uniform(0, 1, n))


def config2(seed=0, n=1_000_000, amp=0.08, octaves=3):
    """1M surfels on a noise-displaced unit icosphere (BASELINE cfg 2)."""
    rng = np.random.default_rng(seed)
    pts, nrm = _displaced_sphere(n, rng, 1.0, amp, octaves, seed + 1)
    ls = rng.uniform(np.log(0.002), np.log(0.01), size=(n, 2))
    alb = 0.5 + 0.45 * np.stack([_value_noise(pts, seed + 10 + c, 3, 3.0) for c in range(3)], axis=1)
    return _raw_cloud(pts, nrm, ls, alb, rng.uniform(0, 1, n), rng.uniform(0, 1, n))


def config3(seed=0, n=500_000, shells=16):
    """16 concentric spheres r in [0.5, 1.5], radial normals, random spin (cfg 3)."""
    rng = np.random.default_rng(seed)
    per = n // shells
    pts = []
    for r in np.linspace(0.5, 1.5, shells):
        d = rng.normal(size=(per, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pts.append(d * r)
    p = np.concatenate(pts)
    m = len(p)
    nrm = p / np.linalg.norm(p, axis=1, keepdims=True)
    cl = _raw_cloud(p, nrm, rng.uniform(np.log(0.004), np.log(0.015), (m, 2)), rng.uniform(0, 1, (m, 3)),
                    rng.uniform(0.1, 0.9, m), rng.uniform(0, 1, m))
    # random rotation about the normal: q_total = q_n * q_z(spin)
    spin = rng.uniform(0, 2 * np.pi, m)
    qz = np.stack([np.cos(spin / 2), np.zeros(m), np.zeros(m), np.sin(spin / 2)], axis=1)
    q = cl["quats"].astype(np.float64)
    w1, x1, y1, z1 = q.T
    w2, x2, y2, z2 = qz.T
    prod = np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=1)
    cl["quats"] = prod.astype(np.float32)
    return cl


def env_lognormal(he, we, seed=0, sigma=1.0):
    """Log-normal HDR environment base radiance (mu=0, sigma)."""
    rng = np.random.default_rng(seed)
    return np.exp(rng.normal(0.0, sigma, (he, we, 3)))


def perturb(cloud, seed=0, pos_sigma=0.01, attr_sigma=0.1):
    """Optimised parameters = ground truth + Gaussian perturbation (cfg 2)."""
    rng = np.random.default_rng(seed)
    out = dict(cloud)
    out["centers"] = (cloud["centers"] + rng.normal(0, pos_sigma, cloud["centers"].shape)).astype(np.float32)
    for k in ("albedo_raw", "metallic_raw", "roughness_raw"):
        out[k] = (cloud[k] + rng.normal(0, attr_sigma, cloud[k].shape)).astype(np.float32)
    return out
