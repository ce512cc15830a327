"""Work statistics of one config-2 view (GPU): rect areas, warp-lane packing
of the record-parallel backward, (8x4 block, record) overlaps of the forward
walk, per-pixel in-rect / covering counts, layer counts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

cloud = ss.SurfelCloud(**scenes.config2(0, 1_000_000))
env = ss.EnvironmentLight.from_base(scenes.env_lognormal(128, 256, 2))
cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[int(os.environ.get("VIEW", "0"))]
res = ss.render(cloud, cam, ss.RenderOptions(with_cover_counts=True), env=env)
st = res.state
keep = st.cull == 0
r = st.records[keep][:, 20:24].contiguous().view(torch.int32).long()
w = r[:, 2] - r[:, 0]
h = r[:, 3] - r[:, 1]
a = (w * h).double()
print(f"kept {int(keep.sum())} pairs {res.stats['pairs']} area sum {a.sum():.4g} mean {a.mean():.2f}")
q = torch.quantile(a[:1000000].float(), torch.tensor([0.1, 0.5, 0.9, 0.99], device=a.device))
print("area p10/50/90/99", q.tolist(), "max", int(a.max()))
for L in (8, 16, 32):
    slots = (torch.ceil(a / L) * L).sum()
    print(f"record-parallel lane packing with {L}-lane groups: {a.sum() / slots:.3f}")
# (8x4 block, record) overlaps
bx0, bx1 = r[:, 0] // 8, (r[:, 2] - 1) // 8
by0, by1 = r[:, 1] // 4, (r[:, 3] - 1) // 4
ov = ((bx1 - bx0 + 1) * (by1 - by0 + 1)).double()
print(f"(8x4 block, record) overlaps {ov.sum():.4g}, in-rect lanes/overlap {a.sum() / ov.sum():.2f}")
for bw, bh in ((4, 8), (16, 2), (4, 4), (8, 8)):
    o2 = (((r[:, 2] - 1) // bw - r[:, 0] // bw + 1) * ((r[:, 3] - 1) // bh - r[:, 1] // bh + 1)).double()
    print(f"  {bw}x{bh} blocks: overlaps {o2.sum():.4g}, in-rect px/overlap {a.sum() / o2.sum():.2f}")
cc = res.cover_counts
if cc is not None:
    print(f"covering evaluations C {cc.double().sum():.4g} ({cc.double().sum() / a.sum():.3f} of rect area)")
nl = res.nlayers.double()
print("layers mean", float(nl.mean()), "max", int(nl.max()), "hist", torch.bincount(res.nlayers.flatten().long()).tolist())
print("alpha>0 px", float((res.alpha > 0).double().mean()))
