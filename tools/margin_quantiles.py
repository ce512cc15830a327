import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_05876_b200 as ss
from paper_2605_05876_b200 import scenes, _lib
from paper_2605_05876_b200.preprocess import run_preprocess
cloud = ss.SurfelCloud(**scenes.config2(0, 1_000_000))
env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 2))
cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[0]
st = run_preprocess(cloud, cam, ss.PreprocessOptions(), _lib.SS_COLOR_IBL, env=env)
keep = st.cull == 0
r = st.records[keep].cpu().numpy()
m = r[:, 19]
rc = r[:, 20:24].view(np.int32)
area = (rc[:, 2] - rc[:, 0]) * (rc[:, 3] - rc[:, 1])
print("inf frac", np.mean(~np.isfinite(m)), "area-weighted inf frac", area[~np.isfinite(m)].sum() / area.sum())
f = m[np.isfinite(m)]
print("finite quantiles 1/10/50/90/99", np.quantile(f, [0.01, 0.1, 0.5, 0.9, 0.99]))
for t in (1e-6, 1e-5, 2e-5, 1e-4, 1e-3):
    sel = np.isfinite(m) & (m <= t)
    print(f"M <= {t:g}: records {sel.mean():.3f}, area share {area[sel].sum() / area.sum():.3f}")
