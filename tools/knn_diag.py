"""Config-4 refinement loop (bench.run_config(4) without the timing): cell
occupancy of the KNN grid and the KNN rebuild time after each refining step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import _lib  # noqa: E402
from paper_2605_05876_b200.densify import DensifyStats  # noqa: E402
from paper_2605_05876_b200.step import TrainStep  # noqa: E402
import bench  # noqa: E402

gt, init, env_base, cams, W, H, extra = bench._config_workload(4)
gt_env = ss.EnvironmentLight.from_base(env_base)
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
del gtc
ts = TrainStep(ss.SurfelCloud(**init), ss.EnvironmentLight(np.log(env_base)), W, H, streams=3,
               surfel_capacity=extra["max_surfels"])
ts.size_pairs(cams[:2])
index = ss.NeighborIndex(ts.cloud, k=8)


def occupancy(cloud):
    n = len(cloud)
    grid, dim = _lib.cell_grid(cloud.centers, n)
    cells = dim ** 3
    starts = grid[16:16 + cells + 1].long()
    cnt = (starts[1:] - starts[:-1])
    occ = cnt[cnt > 0].double()
    # candidate work of the r=1 shell: per query, the points of its 27 cells (upper bound: m * 27 * max)
    return dim, int(occ.numel()), float(occ.mean()), float(occ.max()), float((occ * occ).sum())


for step in range(int(os.environ.get("STEPS", "6"))):
    ts.step(cams, targets)
    st = DensifyStats.zeros(len(ts.cloud))
    st.accumulate(ts.grads["ss_grad"], ts.view_count)
    _, reasons = ts.refine(st, index.mean_dist, extra["max_surfels"], quantile=extra["quantile"])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    index.rebuild(ts.cloud)
    b.record()
    torch.cuda.synchronize()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record()
    index.rebuild(ts.cloud)  # again: allocations cached
    b2.record()
    torch.cuda.synchronize()
    dim, nocc, mean, mx, sq = occupancy(ts.cloud)
    md = index.mean_dist
    short = int((index.neighbors < 0).any(1).sum())
    print(f"step {step}: n {len(ts.cloud)} reasons {reasons} knn {a.elapsed_time(b):.1f} ms (again {a2.elapsed_time(b2):.1f}) | dim {dim} occupied {nocc} "
          f"mean {mean:.1f} max {mx:.0f} sum m^2 {sq:.3g} | short rows {short} mean_dist p50 {float(md.median()):.2e} "
          f"max {float(md.max()):.2e}", flush=True)
