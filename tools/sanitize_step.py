"""A small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): render + both backward paths, a 2-view training step
(L1 and photometric with consolidation), the refinement pass, binning with an
overflowing pair buffer.  Every native kernel of the library runs at least
once at a size the sanitizers finish in minutes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

gt = scenes.config2(0, 3000, amp=0.12, octaves=5)
init = scenes.perturb(gt, 1)
env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 2))
cams = ss.fibonacci_cameras(2, 3.0, 96, 80, fov_y_deg=40.0)
cloud = ss.SurfelCloud(**init)
targets = [ss.render(ss.SurfelCloud(**gt), c, ss.RenderOptions(), env=env).rgb.contiguous() for c in cams]
res = ss.render(cloud, cams[0], ss.RenderOptions(with_cover_counts=True, collect_stacks=True), env=env)
g = torch.randn_like(res.rgb)
for path in ("records", "walk"):
    ss.backward_image(cloud, res, g_rgb=g, cons_scale=1e-3, path=path)
ts = ss.TrainStep(cloud, env, 96, 80, pair_capacity=500, surfel_capacity=3300)  # overflow -> regrow
ts.step(cams, targets)
tp = ss.TrainStep(ss.SurfelCloud(**init), env, 96, 80, loss="photometric", cons_scale=1e-4)
tp.step(cams, targets, masks=[torch.ones(80, 96, device="cuda")] * 2)
stats = ss.DensifyStats.zeros(len(ts.cloud))
stats.accumulate(ts.grads["ss_grad"], ts.view_count)
idx = ss.NeighborIndex(ts.cloud, k=8)
ts.refine(stats, idx.mean_dist, 3150, quantile=0.95)
ts.step(cams, targets)
torch.cuda.synchronize()
print("sanitize workload ok", len(ts.cloud), ts.regrows)
