"""Timing of the refinement scan pieces on config 2 (KNN index, prune, split)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes, densify  # noqa: E402

cloud = ss.SurfelCloud(**scenes.config2(0, 1_000_000))
n = len(cloud)
st = densify.DensifyStats.zeros(n)
g = torch.rand(n, device="cuda", dtype=torch.float64) * 1e-3
st.accumulate(g, torch.ones(n, device="cuda", dtype=torch.bool))


def t(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms")
    return out


knn = t("NeighborIndex(k=8)", lambda: ss.NeighborIndex(cloud, k=8))
t("prune_keep_mask", lambda: densify.prune_keep_mask(cloud, st))
t("refine_topology", lambda: densify.refine_topology(cloud, st, knn.mean_dist, int(1.05 * n)))
