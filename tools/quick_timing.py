import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_05876_b200 as ss
from paper_2605_05876_b200 import scenes
t0=time.time()
cl = scenes.config2(0)
print("gen", time.time()-t0, flush=True)
cloud = ss.SurfelCloud(**cl)
env = ss.EnvironmentLight.from_base(scenes.env_lognormal(128, 256, 1))
cams = ss.fibonacci_cameras(int(os.environ.get("QT_VIEWS", "8")), 3.5, 800, 800)
opt = ss.RenderOptions()
g = torch.randn(800,800,3, device="cuda")*1e-6
for it in range(int(os.environ.get("QT_ITERS", "2"))):
    for cam in cams:
        torch.cuda.synchronize(); t=time.time()
        res = ss.render(cloud, cam, opt, env=env)
        torch.cuda.synchronize(); t1=time.time()
        back = ss.backward_image(cloud, res, g_rgb=g)
        torch.cuda.synchronize(); t2=time.time()
        if it==1: print(f"P={res.stats['pairs']} Nk={res.stats['surfels_rasterized']} fwd(api) {1e3*(t1-t):.2f} ms bwd(api) {1e3*(t2-t1):.2f} ms maxlayers {int(res.nlayers.max())}", flush=True)
