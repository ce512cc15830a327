"""Profiling driver: the bench.py workload (config 2, 1M surfels, 800^2),
one warm-up step then NVIEWS views of one step inside an NVTX range
"ss_step" so ncu can filter with --nvtx --nvtx-include ss_step/."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import TrainStep  # noqa: E402

NV = int(os.environ.get("NVIEWS", "8"))
gt = scenes.config2(0, 1_000_000)
init = scenes.perturb(gt, 1)
env_base = scenes.env_lognormal(128, 256, 2)
cams = ss.fibonacci_cameras(64, 3.5, 800, 800)[:NV]
gt_env = ss.EnvironmentLight.from_base(env_base)
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
del gtc
cloud = ss.SurfelCloud(**init)
env = ss.EnvironmentLight(np.log(env_base))
ts = TrainStep(cloud, env, 800, 800)
ts.size_pairs(cams[:2])
ts.step(cams, targets)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("ss_step")
ts.step(cams, targets)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("profile step ok", float(ts.loss_f.item()))
