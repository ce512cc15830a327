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
print("inf frac", np.mean(~np.isfinite(m)))
f = m[np.isfinite(m)]
if len(f): print("finite quantiles", np.quantile(f, [0.1, 0.5, 0.9, 0.99]))
# a typical record
i = np.where(np.isfinite(m))[0][:1] if len(f) else [0]
np.set_printoptions(precision=6, suppress=False)
print("t1 t2 t4 sinv", r[0, :12], "rect", r[0, 20:24].view(np.int32))
# reasons for an infinite margin, replicated in float64 numpy
e = 2.0 ** -24
T1, T2, T4 = r[:, 0:3].astype(np.float64), r[:, 3:6].astype(np.float64), r[:, 6:9].astype(np.float64)
S0, S1, S2 = r[:, 9].astype(np.float64), r[:, 10].astype(np.float64), r[:, 11].astype(np.float64)
rc = r[:, 20:24].view(np.int32)
W = H = 800
ndx = lambda ix: ((ix + 0.5) * (2.0 / W) - 1.0).astype(np.float32).astype(np.float64)
ndy = lambda iy: (1.0 - (iy + 0.5) * (2.0 / H)).astype(np.float32).astype(np.float64)
xs = [ndx(rc[:, 0]), ndx(rc[:, 2] - 1)]
ys = [ndy(rc[:, 1]), ndy(rc[:, 3] - 1)]
dens = []
for x in xs:
    for y in ys:
        k = x[:, None] * T4 - T1
        l = y[:, None] * T4 - T2
        dens.append(k[:, 0] * l[:, 1] - k[:, 1] * l[:, 0])
dens = np.stack(dens, 1)
sign_change = ~((dens > 0).all(1) | (dens < 0).all(1))
print("den sign change frac", sign_change.mean(), " among inf:", sign_change[~np.isfinite(m)].mean())
area = (rc[:, 2] - rc[:, 0]) * (rc[:, 3] - rc[:, 1])
print("inf by area quantile: median area all", np.median(area), "median area inf", np.median(area[~np.isfinite(m)]))
det = S0 * S2 - S1 ** 2
print("sinv det<=0 frac", (det <= 0).mean())
