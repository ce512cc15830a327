"""On-disk formats against files written by the
reference's own sceneio (tests/golden/make_golden_io.py).  GPU-marked because
the loaders build device SurfelClouds."""

import json
import os

import numpy as np
import pytest
import torch

from parity import host

pytestmark = pytest.mark.gpu

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import sceneio  # noqa: E402

IO = os.path.join(os.path.dirname(__file__), "golden", "io")
KEYS = ("centers", "quats", "log_scales", "albedo_raw", "metallic_raw", "roughness_raw")


def test_scene_round_trips_with_reference_files(tmp_path):
    ref = np.load(os.path.join(IO, "scene.npz"))
    cloud, env = sceneio.load_scene(os.path.join(IO, "scene.npz"))
    for k in KEYS:
        np.testing.assert_array_equal(host(getattr(cloud, k)), ref[k])
    assert env.levels == int(ref["env_levels"])
    np.testing.assert_allclose(host(env.base_log), ref["env_base_log"], rtol=1e-6)
    out = tmp_path / "scene.npz"
    sceneio.save_scene(out, cloud, env)
    got = np.load(out)
    assert set(got.files) == set(ref.files)
    for k in KEYS + ("scene_version", "env_levels"):
        assert got[k].dtype == ref[k].dtype
        np.testing.assert_array_equal(got[k], ref[k])


def test_checkpoint_loads_into_the_device_optimizer(tmp_path):
    cloud, env, opt_arrays, step, nb, md, extra = sceneio.load_checkpoint(os.path.join(IO, "checkpoint.npz"))
    assert step == 17 and nb.shape == (50, 4) and md.shape == (50,)
    np.testing.assert_array_equal(extra["note"], np.arange(3))
    opt = ss.Adam()
    opt.load_state_arrays(opt_arrays)
    assert set(opt.m) == set(KEYS) and all(opt.t[k] == 1 for k in KEYS)
    np.testing.assert_allclose(host(opt.m["centers"]), opt_arrays["adam_m_centers"], rtol=1e-6)
    out = tmp_path / "ck.npz"
    sceneio.save_checkpoint(out, cloud, env, opt, step, nb, md, extra=extra)
    back = sceneio.load_checkpoint(out)
    assert back[3] == 17
    np.testing.assert_array_equal(back[4], nb)
    for k in KEYS:
        np.testing.assert_array_equal(host(getattr(back[0], k)), host(getattr(cloud, k)))
    with pytest.raises(sceneio.SceneFormatError):
        sceneio.load_scene(out)  # a checkpoint is not a scene file


def test_ply_matches_reference_writer_and_reader(tmp_path):
    cloud, _ = sceneio.load_scene(os.path.join(IO, "scene.npz"))
    out = tmp_path / "cloud.ply"
    sceneio.export_ply(out, cloud)
    ours, theirs = out.read_bytes(), open(os.path.join(IO, "cloud.ply"), "rb").read()
    split = theirs.index(b"end_header\n") + len(b"end_header\n")
    assert ours[:split] == theirs[:split]
    a = np.frombuffer(ours[split:], "<f4")
    b = np.frombuffer(theirs[split:], "<f4")
    np.testing.assert_allclose(a, b, rtol=2e-6, atol=1e-7)
    ref = np.load(os.path.join(IO, "ref.npz"))
    back = sceneio.import_ply(os.path.join(IO, "cloud.ply"))
    for k in KEYS:
        np.testing.assert_array_equal(host(getattr(back, k)), ref[f"ply_{k}"])
    bad = tmp_path / "bad.ply"
    bad.write_bytes(theirs[:split + 10])
    with pytest.raises(sceneio.SceneFormatError):
        sceneio.import_ply(bad)


def test_datasets_load_like_the_reference(tmp_path):
    ds = sceneio.load_dataset(os.path.join(IO, "ds", "dataset.json"))
    desc = json.load(open(os.path.join(IO, "ds", "dataset.json")))
    assert ds["extent"] == 1.5 and len(ds["cameras"]) == 2
    for i, fr in enumerate(desc["frames"]):
        np.testing.assert_array_equal(ds["cameras"][i].view, np.asarray(fr["view"]))
        np.testing.assert_array_equal(ds["images"][i], np.load(os.path.join(IO, "ds", fr["image"])))
        np.testing.assert_array_equal(ds["masks"][i], np.load(os.path.join(IO, "ds", fr["mask"])))
    ref = np.load(os.path.join(IO, "ref.npz"))
    tf = sceneio.load_dataset(os.path.join(IO, "tf", "transforms.json"))
    for i in range(2):
        np.testing.assert_allclose(tf["cameras"][i].view, ref[f"tf_view_{i}"], rtol=1e-12, atol=1e-15)
        np.testing.assert_array_equal(tf["cameras"][i].proj, ref[f"tf_proj_{i}"])
        np.testing.assert_array_equal(tf["images"][i], ref[f"tf_img_{i}"])
        np.testing.assert_array_equal(tf["masks"][i], ref[f"tf_mask_{i}"])
    # our writer -> our reader round trip, device images accepted
    p = sceneio.save_dataset(tmp_path / "d2", ds["cameras"], [torch.as_tensor(im, device="cuda") for im in ds["images"]],
                             ds["masks"], extent=2.0)
    d2 = sceneio.load_dataset(p)
    np.testing.assert_array_equal(d2["images"][1], ds["images"][1])
    with pytest.raises(sceneio.SceneFormatError):
        sceneio.load_image(tmp_path / "x.tiff")
