"""One photometric-loss step (NVTX ss_step) of NVIEWS config-2 views for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import TrainStep  # noqa: E402

NV = int(os.environ.get("NVIEWS", "4"))
gt = scenes.config2(0, 1_000_000)
env_base = scenes.env_lognormal(128, 256, 2)
cams = ss.fibonacci_cameras(64, 3.5, 800, 800)[:NV]
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=ss.EnvironmentLight.from_base(env_base)).rgb.contiguous()
           for c in cams]
cloud = ss.SurfelCloud(**scenes.perturb(gt, 1))
ts = TrainStep(cloud, ss.EnvironmentLight(np.log(env_base)), 800, 800, loss="photometric", streams=1)
ts.size_pairs(cams[:2])
ts.step(cams, targets)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("ss_step")
ts.step(cams, targets)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", float(ts.loss_f.item()))
