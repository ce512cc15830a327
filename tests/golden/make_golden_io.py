"""Golden files for the on-disk formats, written by the
REFERENCE's own sceneio (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py

Writes tests/golden/io/: scene.npz (with env), checkpoint.npz (Adam state,
KNN table, extras), cloud.ply, a two-view dataset (dataset.json + .npy images
and masks), a transforms.json dataset with RGBA .png images, and ref.npz
holding the arrays the reference loads back from each of them.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_cache")
os.environ.setdefault("SURFSPLAT_CACHE_DIR", "/tmp/ss_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from surfsplat import sceneio  # noqa: E402
from surfsplat.adam import Adam  # noqa: E402
from surfsplat.camera import Camera  # noqa: E402
from surfsplat.knn import NeighborIndex  # noqa: E402
from surfsplat.shading import EnvironmentLight  # noqa: E402
from surfsplat.surfels import SurfelCloud  # noqa: E402

KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(5)
    n = 50
    cloud = SurfelCloud(centers=rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                        quats=rng.normal(size=(n, 4)).astype(np.float32),
                        log_scales=np.log(rng.uniform(0.01, 0.05, (n, 2))).astype(np.float32),
                        albedo_raw=rng.normal(size=(n, 3)).astype(np.float32),
                        metallic_raw=rng.normal(size=n).astype(np.float32),
                        roughness_raw=rng.normal(size=n).astype(np.float32))
    env = EnvironmentLight.from_base(np.exp(rng.normal(0, 1, (8, 16, 3))), levels=4)
    ref = {}
    sceneio.save_scene(os.path.join(OUT, "scene.npz"), cloud, env)
    opt = Adam()
    for k in KEYS:
        opt.step(k, getattr(cloud, k).astype(np.float64).copy(), rng.normal(size=getattr(cloud, k).shape), 1e-3)
    idx = NeighborIndex(cloud, k=4)
    sceneio.save_checkpoint(os.path.join(OUT, "checkpoint.npz"), cloud, env, opt, 17, idx.neighbors, idx.mean_dist,
                            extra={"note": np.arange(3)})
    sceneio.export_ply(os.path.join(OUT, "cloud.ply"), cloud)
    back = sceneio.import_ply(os.path.join(OUT, "cloud.ply"))
    for k in KEYS:
        ref[f"ply_{k}"] = getattr(back, k)
    cams = [Camera.perspective(24, 16, 40.0, (2.0, 0.5 * i, 1.0), (0, 0, 0)) for i in range(2)]
    imgs = [rng.uniform(0, 2, (16, 24, 3)).astype(np.float32) for _ in cams]
    masks = [(rng.uniform(size=(16, 24)) > 0.5).astype(np.float32) for _ in cams]
    sceneio.save_dataset(os.path.join(OUT, "ds"), cams, imgs, masks, extent=1.5)
    # transforms.json with RGBA png images
    os.makedirs(os.path.join(OUT, "tf"), exist_ok=True)
    frames = []
    for i in range(2):
        rgba = np.concatenate([rng.uniform(0, 1, (12, 20, 3)), (rng.uniform(size=(12, 20, 1)) > 0.5)], axis=2)
        sceneio.write_png(os.path.join(OUT, "tf", f"r_{i}.png"), rgba)
        c2w = np.linalg.inv(cams[i].view)
        frames.append({"file_path": f"r_{i}", "transform_matrix": c2w.tolist()})
    with open(os.path.join(OUT, "tf", "transforms.json"), "w") as fh:
        json.dump({"camera_angle_x": 0.7, "frames": frames}, fh)
    tf = sceneio.load_dataset(os.path.join(OUT, "tf", "transforms.json"))
    for i in range(2):
        ref[f"tf_view_{i}"] = tf["cameras"][i].view
        ref[f"tf_proj_{i}"] = tf["cameras"][i].proj
        ref[f"tf_img_{i}"] = tf["images"][i]
        ref[f"tf_mask_{i}"] = tf["masks"][i]
    np.savez_compressed(os.path.join(OUT, "ref.npz"), **ref)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
