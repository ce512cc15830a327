"""Per-stage device times of the bench workload (config 2) with ONE worker
stream (no overlap: each stage timed alone by CUDA events), then whole-step
views/s for 1, 2 and 3 worker streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import TrainStep  # noqa: E402

NV = int(os.environ.get("NVIEWS", "16"))
gt = scenes.config2(0, 1_000_000)
if os.environ.get("MORTON"):  # spatially coherent surfel order (study)
    perm = scenes.morton_order(gt["centers"])
    gt = {k: v[perm] for k, v in gt.items()}
init = scenes.perturb(gt, 1)
env_base = scenes.env_lognormal(128, 256, 2)
cams = ss.fibonacci_cameras(64, 3.5, 800, 800)[:NV]
gt_env = ss.EnvironmentLight.from_base(env_base)
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
del gtc
cloud = ss.SurfelCloud(**init)
env = ss.EnvironmentLight(np.log(env_base))
LOSS = os.environ.get("LOSS", "l1")
for S in tuple(int(v) for v in os.environ.get("STREAMS", "1,2,3").split(",")):
    ts = TrainStep(cloud, env, 800, 800, streams=S, loss=LOSS, tile=int(os.environ.get("TILE", "16")))
    ts.size_pairs(cams[:2])
    for _ in range(2):
        ts.step(cams, targets)
    torch.cuda.synchronize()
    if S == 1:
        ts.kernel_events = []
        ts.step(cams, targets)
        torch.cuda.synchronize()
        per = {}
        for name, a, b in ts.kernel_events:
            per.setdefault(name, []).append(a.elapsed_time(b))
        ts.kernel_events = None
        tot = 0.0
        for k, v in per.items():
            print(f"  {k:16s} {np.mean(v):7.3f} ms/view")
            tot += np.mean(v)
        print(f"  {'sum':16s} {tot:7.3f} ms/view")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ts.step(cams, targets)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"streams={S}: step {ms:.2f} ms for {NV} views -> {NV / ms * 1e3:.1f} views/s ({ms / NV:.3f} ms/view)")
    del ts
    torch.cuda.empty_cache()
