"""Eager vs CUDA-graph step times (TrainStep.step(graph=...)) on BASELINE
configs 0, 1 and 2, and the gradient agreement of the two."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import PARAMS, TrainStep  # noqa: E402


def workload(cfg):
    if cfg == 2:
        gt = scenes.config2(0, 1_000_000)
        return gt, scenes.perturb(gt, 1), scenes.env_lognormal(128, 256, 2), ss.fibonacci_cameras(64, 3.5, 800, 800), \
            800, 800
    gt, init, env_base, cams, W, H, _ = bench._config_workload(cfg)
    return gt, init, env_base, cams, W, H


for cfg in (0, 1, 2):
    gt, init, env_base, cams, W, H = workload(cfg)
    gtc = ss.SurfelCloud(**gt)
    gt_env = ss.EnvironmentLight.from_base(env_base)
    targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
    del gtc
    res = {}
    for graph in (False, True):
        cloud = ss.SurfelCloud(**init)
        env = ss.EnvironmentLight(np.log(env_base))
        ts = TrainStep(cloud, env, W, H, streams=int(os.environ.get("STREAMS", "3")))
        ts.size_pairs(cams[:2])
        ts.gradients_graphed(cams, targets) if graph else ts.gradients(cams, targets)
        g0 = {k: ts.grads[k].clone() for k in PARAMS}
        if graph:  # replayed gradients vs the eager pass's
            ts.gradients_graphed(cams, targets)
            err = max(float((ts.grads[k] - g0[k]).abs().max() / g0[k].abs().max().clamp_min(1e-30)) for k in PARAMS)
            print(f"config{cfg}: replay vs eager gradients, max |diff| / max|g| = {err:.2e}")
        for _ in range(3):
            ts.step(cams, targets, graph=graph)
        torch.cuda.synchronize()
        n = 20 if cfg < 2 else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            ts.step(cams, targets, graph=graph)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        res[graph] = ms
        print(f"config{cfg} graph={graph}: {ms:.3f} ms/step, {len(cams) / ms * 1e3:.1f} views/s")
        del ts
        torch.cuda.empty_cache()
