"""Diagnose gradient outliers of the config-2 training step vs the oracle:
for the worst surfels, compare the record path, the walk path and the oracle,
and print the surfel's rect, covering pixels and accumulator channels."""

import sys
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2605_05876_b200 as ss  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import PARAMS, TrainStep  # noqa: E402
from parity import grad_outliers  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    if cfg == "3":
        gt = scenes.config3(0, 500_000)
        base_log = np.log(scenes.env_lognormal(64, 128, 3))
        R = 1024
        cam = ss.fibonacci_cameras(16, 3.5, R, R)[3]
    else:
        gt = scenes.config2(0, 1_000_000)
        base_log = np.log(scenes.env_lognormal(128, 256, 2))
        R = 800
        cam = ss.fibonacci_cameras(64, 3.5, R, R)[5]
    opt = scenes.perturb(gt, 1)
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    ts = TrainStep(cloud, env, R, R)
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    oenv = O.EnvOracle(base_log.astype(np.float32).astype(np.float64) if "--f32env" in sys.argv else base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    rgb = ts.captured_rgb[-1].cpu().numpy().astype(np.float64)
    g = np.sign(rgb - target.cpu().numpy()) / rgb.size
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    gt_ = torch.tensor(g, device="cuda", dtype=torch.float32)
    walk = ss.backward_image(cloud, res, g_rgb=gt_, path="walk")
    rec = ss.backward_image(cloud, res, g_rgb=gt_, path="records")
    bad_surfels = set()
    for k in PARAMS:
        w = ts.grads[k].shape[1] if ts.grads[k].dim() > 1 else 1
        outl, n = grad_outliers(ts.grads[k], og[k])
        print(k, "step outliers", n)
        for o in outl:
            bad_surfels.add(o[0] // w)
        for name, b in (("walk", walk), ("records", rec)):
            outl2, n2 = grad_outliers(getattr(b, k).reshape(ts.grads[k].shape), og[k])
            print("   ", name, "outliers", n2, [o[0] // w for o in outl2][:8])
    recs = res.state.records.cpu().numpy()
    rects = recs[:, 20:24].view(np.int32)
    for i in sorted(bad_surfels):
        r = rects[i]
        area = (r[2] - r[0]) * (r[3] - r[1])
        print(f"surfel {i}: rect {r.tolist()} area {area} margin {recs[i, 19]:.3g} t4z {recs[i, 8]:.4g} "
              f"view_z {recs[i, 13]:.4g} covered {int(rec.touch_count[i])}")
        for k in ("centers", "log_scales", "quats"):
            print("   ", k, "step", ts.grads[k][i].cpu().numpy(), "walk",
                  getattr(walk, k).reshape(ts.grads[k].shape)[i].cpu().numpy(), "records",
                  getattr(rec, k).reshape(ts.grads[k].shape)[i].cpu().numpy(), "oracle", og[k][i])
        print("    ss", float(ts.grads["ss_grad"][i]), float(og["ss_grad"][i]))


if __name__ == "__main__" and "--colours" not in sys.argv and "--records" not in sys.argv:
    main()


def colour_probe():
    """Is the residual log-scale error colour-driven?  Oracle backward with
    the B200 colours (explicit) vs with its own float64-shaded colours."""
    gt = scenes.config2(0, 1_000_000)
    base_log = np.log(scenes.env_lognormal(128, 256, 2))
    cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[5]
    opt = scenes.perturb(gt, 1)
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    cols = res.colors.cpu().numpy()
    oenv = O.EnvOracle(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    ocols = ores.colors if hasattr(ores, "colors") else None
    if ocols is not None:
        d = cols != ocols.astype(np.float32)
        print("colour entries differing from the oracle's:", int(d.sum()), "of", d.size,
              "max rel", float(np.max(np.abs(cols - ocols) / np.maximum(np.abs(ocols), 1e-30))))
    rgb = res.rgb.cpu().numpy().astype(np.float64)
    g = np.sign(rgb - target.cpu().numpy()) / rgb.size
    ores_e = O.render(co, cam, colors=cols)
    og_e = O.backward_image(co, ores_e, g, None, 0.0)
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
    back = ss.backward_image(cloud, res, g_rgb=torch.tensor(g, device="cuda", dtype=torch.float32))
    for i in (885527, 714081, 659573, 589042):
        print(i, "ours", back.log_scales[i].cpu().numpy(), "oracle(ibl)", og["log_scales"][i],
              "oracle(our colours)", og_e["log_scales"][i])


if __name__ == "__main__" and "--colours" in sys.argv:
    colour_probe()


def _moments_to_rows(a, rec):
    """acc row in the centred-moment layout -> dL/dt1, dt2, dt4 (float64)."""
    t1, t2, t4 = rec[0:3].astype(np.float64), rec[3:6].astype(np.float64), rec[6:9].astype(np.float64)
    cx = np.float32(rec[2]) / np.float32(rec[8])
    cy = np.float32(rec[5]) / np.float32(rec[8])
    S = a[0:3].astype(np.float64)
    Sx = a[3:6].astype(np.float64) + float(cx) * S
    Sy = a[6:9].astype(np.float64) + float(cy) * S
    g1 = np.cross(t2, S) - np.cross(t4, Sy)
    g2 = np.cross(S, t1) - np.cross(Sx, t4)
    g4 = np.cross(t1, Sy) - np.cross(t2, Sx)
    return np.concatenate([g1, g2, g4])


def record_probe():
    """Per-record accumulator rows (17 channels before the per-surfel chain)
    of the training step vs the oracle's merged pair rows."""
    if "3" in sys.argv:
        gt = scenes.config3(0, 500_000)
        base_log = np.log(scenes.env_lognormal(64, 128, 3))
        R = 1024
        cam = ss.fibonacci_cameras(16, 3.5, R, R)[3]
        probe = (443082, 479913, 480338)
    else:
        gt = scenes.config2(0, 1_000_000)
        base_log = np.log(scenes.env_lognormal(128, 256, 2))
        R = 800
        cam = ss.fibonacci_cameras(64, 3.5, R, R)[5]
        probe = (885527, 714081, 659573, 589042, 443082)
    opt = scenes.perturb(gt, 1)
    env = ss.EnvironmentLight(base_log)
    target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
    cloud = ss.SurfelCloud(**opt)
    photo = "--photometric" in sys.argv
    ts = TrainStep(cloud, env, R, R, streams=1, loss="photometric" if photo else "l1")
    ts.captured_rgb = []
    ts.gradients([cam], [target])
    acc = ts.bufs[0].acc.cpu().numpy()
    recs = ts.bufs[0].records.cpu().numpy()
    oenv = O.EnvOracle(base_log)
    co = SimpleNamespace(**opt)
    ores = O.render(co, cam, env=oenv)
    rgb = ts.captured_rgb[-1].cpu().numpy().astype(np.float64)
    if photo:
        tg = target.cpu().numpy().astype(np.float64)
        _, gm = O.photometric_loss(O.tone_map(rgb, "hdr-loss"), O.tone_map(tg, "hdr-loss"), 0.2)
        g = O.tone_map_backward(rgb, "hdr-loss", gm)
        probe = tuple(int(a) for a in sys.argv[sys.argv.index("--photometric") + 1].split(","))
        g64 = ts.bufs[0].g_rgb64.cpu().numpy()
        d = np.abs(g64 - g)
        print("image gradient: max |g64 - oracle|", d.max(), "max |oracle|", np.abs(g).max(),
              "max rel", (d / np.maximum(np.abs(g), 1e-300)).max())
    else:
        g = np.sign(rgb - target.cpu().numpy()) / rgb.size
    og = O.backward_image(co, ores, g, None, 0.0, env=oenv, return_records=True)
    src = ores.proj["source_index"]
    pos = {int(s): k for k, s in enumerate(src)}
    np.set_printoptions(precision=9, linewidth=200)
    for i in probe:
        k = pos[i]
        a = acc[i].astype(np.float64)
        if a[19] == 2.0:  # big record: float64 rows in acc64 (T-row layout)
            r = ts.bufs[0].acc64[int(acc[i][0].view(np.int32))].cpu().numpy()
            a[0:17] = r[0:17]
            print("   (big record, float64 rows; gz", r[17], ")")
        elif a[19] == 1.0:
            a[0:9] = _moments_to_rows(a, recs[i])
        print(i, "layout", a[19], "touch", acc[i][18].view(np.int32),
              "oracle touch", og["touch_rec"][k])
        print("   ours  ", a[:17], "ss", a[17])
        print("   oracle", og["records"][k], "ss", og["ss_rec"][k])
        o = np.asarray(og["records"][k], np.float64)
        print("   rel   ", np.abs(a[:17] - o) / np.maximum(np.abs(o), 1e-30))
        rr = recs[i]
        pj = ores.proj
        ours = {"t1": rr[0:3], "t2": rr[3:6], "t4": rr[6:9], "sinv": rr[9:12], "n_f": rr[12:13], "view_z": rr[13:14],
                "z_start": rr[14:15], "z_end": rr[15:16], "color": rr[16:19], "rect": rr[20:24].view(np.int32)}
        for key, val in ours.items():
            if key == "color":
                ref = np.asarray(ores.colors)[i] if hasattr(ores, "colors") else None
            else:
                ref = np.asarray(pj[key])[k] if key in pj else None
            print("   ", key, val, "oracle", ref)


if __name__ == "__main__" and "--records" in sys.argv:
    record_probe()
