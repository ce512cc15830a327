"""Device-resident step() vs step_host() (pinned host targets, copies inside
the step) on the bench workload with NVIEWS views, for copy lookaheads 1..3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import TrainStep  # noqa: E402

NV = int(os.environ.get("NVIEWS", "32"))
gt = scenes.config2(0, 1_000_000)
init = scenes.perturb(gt, 1)
env_base = scenes.env_lognormal(128, 256, 2)
cams = ss.fibonacci_cameras(64, 3.5, 800, 800)[:NV]
gt_env = ss.EnvironmentLight.from_base(env_base)
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
host = [t.cpu().pin_memory() for t in targets]
del gtc
ts = TrainStep(ss.SurfelCloud(**init), ss.EnvironmentLight(np.log(env_base)), 800, 800, streams=3)
ts.size_pairs(cams[:4])


def timed(fn, steps=3):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return NV / (a.elapsed_time(b) / steps / 1e3)


print(f"resident step: {timed(lambda: ts.step(cams, targets)):.1f} views/s")
for la in (1, 2, 3):
    ts.copy_lookahead = la
    print(f"step_host lookahead {la}: {timed(lambda: ts.step_host(cams, host).item()):.1f} views/s")
print(f"resident step: {timed(lambda: ts.step(cams, targets)):.1f} views/s")
