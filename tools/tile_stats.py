"""Per-tile pair-list lengths of one config-2 view (GPU): the forward walk's
per-warp cost is proportional to its tile's list, so the heaviest tiles set
the launch's tail."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402

cloud = ss.SurfelCloud(**scenes.config2(0, 1_000_000))
env = ss.EnvironmentLight.from_base(scenes.env_lognormal(128, 256, 2))
for v in (0, 17, 40):
    cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[v]
    res = ss.render(cloud, cam, ss.RenderOptions(), env=env)
    off = res.tile_offsets.long()
    c = (off[1:] - off[:-1]).double()
    s, _ = torch.sort(c, descending=True)
    tot = c.sum()
    print(f"view {v}: tiles {len(c)} pairs {tot:.4g} mean {c.mean():.1f} max {s[0]:.0f} "
          f"top10 {[int(x) for x in s[:10].tolist()]}")
    print("   quantiles p50/p90/p99", torch.quantile(c.float(), torch.tensor([0.5, 0.9, 0.99], device=c.device)).tolist(),
          f" max/mean {s[0] / c.mean():.1f}  share of top 1% {s[:len(c) // 100].sum() / tot:.3f}")
