"""Record-path backward of one config-2 view (touch counts + gradients) saved
for comparing builds: python tools/bwd_compare.py OUT.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

gt = scenes.config2(0, 1_000_000)
cloud = ss.SurfelCloud(**scenes.perturb(gt, 1))
env = ss.EnvironmentLight(np.log(scenes.env_lognormal(128, 256, 2)))
out = {}
for v in (3, 11, 40):
    cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[v]
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    g = torch.tensor(np.random.default_rng(v).normal(0, 1e-6, (800, 800, 3)), device="cuda", dtype=torch.float32)
    b = ss.backward_image(cloud, res, g_rgb=g)
    out[f"touch_{v}"] = b.touch_count.cpu().numpy()
    out[f"centers_{v}"] = b.centers.cpu().numpy()
    out[f"ss_{v}"] = b.ss_grad.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
