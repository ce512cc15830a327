import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_05876_b200 as ss
from paper_2605_05876_b200 import scenes
from paper_2605_05876_b200.preprocess import run_preprocess
cloud = ss.SurfelCloud(**scenes.config2(0, 1_000_000))
env = ss.EnvironmentLight.from_base(scenes.env_lognormal(16, 32, 2))
cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[0]
st = run_preprocess(cloud, cam, ss.PreprocessOptions(), 1, env=env)
r = st.records[st.cull == 0][:, 20:24].contiguous().view(torch.int32).cpu().numpy()
w = r[:, 2] - r[:, 0]; h = r[:, 3] - r[:, 1]; a = w * h
print("kept", len(a), "area mean", a.mean(), "p50/p90/p99/max", np.percentile(a, [50, 90, 99]), a.max())
for th in (256, 512, 2048, 10000):
    m = a > th
    print(f"> {th}: n={m.sum()} total area {a[m].sum()} ({a[m].sum()/a.sum()*100:.1f}% of all)")
big = np.argsort(-a)[:5]
print("biggest w,h:", list(zip(w[big], h[big])))
rec = st.records[st.cull == 0].cpu().numpy()[big]
print("n_f of biggest", rec[:, 12], "sinv", rec[:, 9:12])
