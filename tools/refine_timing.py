"""Timing of the refinement pass pieces (KNN index, isolation, the fused
refine_topology) at 1M (config 2) and 4M (config 4 geometry) surfels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes, densify  # noqa: E402


def t(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{name:34s} {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms", flush=True)
    return out


for n, amp, oct_ in ((1_000_000, 0.08, 3), (4_000_000, 0.12, 5)):
    cloud = ss.SurfelCloud(**scenes.config2(0, n, amp=amp, octaves=oct_))
    st = densify.DensifyStats.zeros(n)
    g = torch.rand(n, device="cuda", dtype=torch.float64) * 1e-3
    st.accumulate(g, torch.ones(n, device="cuda", dtype=torch.bool))
    print(f"--- {n} surfels")
    knn = t("NeighborIndex(k=8)", lambda: ss.NeighborIndex(cloud, k=8))
    t("isolated_flags", lambda: densify.isolated_flags(cloud))
    t("refine_topology (device)", lambda: densify.refine_topology(cloud, st, knn.mean_dist, int(1.05 * n),
                                                                 quantile=0.95))
