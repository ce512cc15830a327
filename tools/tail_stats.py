"""Tail analysis of the two rasterisers (library built with -DSS_CTA_TIMING):
per-CTA (forward) and per-warp (record backward) start/end timestamps of one
config-2 view run alone, turned into the number of active CTAs / warps over
the launch and the time spent with few of them left."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import _lib, scenes  # noqa: E402
from paper_2605_05876_b200.step import TrainStep  # noqa: E402

gt = scenes.config2(0, 1_000_000)
init = scenes.perturb(gt, 1)
env_base = scenes.env_lognormal(128, 256, 2)
cams = ss.fibonacci_cameras(64, 3.5, 800, 800)[:2]
gt_env = ss.EnvironmentLight.from_base(env_base)
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
del gtc
ts = TrainStep(ss.SurfelCloud(**init), ss.EnvironmentLight(np.log(env_base)), 800, 800, streams=1)
ts.size_pairs(cams)
ts.step(cams, targets)
lib = _lib.load()
fb = torch.zeros(3 * 50 * 50 * 4, device="cuda", dtype=torch.int64)
bb = torch.zeros(3 * 148 * 3 * 8 * 2, device="cuda", dtype=torch.int64)
_lib.check(lib.ss_debug_set_fwd_timing(_lib.ptr(fb)), "set_fwd_timing")
_lib.check(lib.ss_debug_set_bwd_timing(_lib.ptr(bb)), "set_bwd_timing")
ts.step(cams[:1], targets[:1])
torch.cuda.synchronize()
lib.ss_debug_set_fwd_timing(None)
lib.ss_debug_set_bwd_timing(None)


def report(name, buf):
    a = buf.view(-1, 3).cpu().numpy()
    a = a[a[:, 1] > 0]
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3  # us
    span = en.max()
    grid = np.linspace(0, span, 401)
    act = np.array([((st <= t) & (en > t)).sum() for t in grid])
    peak = act.max()
    busy = (en - st).sum()
    print(f"{name}: units {len(a)} span {span:.1f} us, peak active {peak}, mean active {act.mean():.1f} "
          f"({act.mean() / peak:.2f} of peak)")
    for f in (0.9, 0.75, 0.5, 0.25, 0.1):
        below = grid[act < f * peak]
        below = below[below > grid[np.argmax(act)]]
        print(f"   time with < {f:.2f} of peak active (after the peak): {(span - below.min()) if len(below) else 0:.1f} us")
    d = en - st
    print(f"   unit duration us: mean {d.mean():.1f} p50 {np.median(d):.1f} p90 {np.percentile(d, 90):.1f} "
          f"max {d.max():.1f}; busy/(span*peak) {busy / (span * peak):.2f}")


report("raster_fwd (per CTA)", fb)
report("splat_bwd (per warp)", bb)
