import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from types import SimpleNamespace
import numpy as np, torch
import paper_2605_05876_b200 as ss
from paper_2605_05876_b200 import scenes
from paper_2605_05876_b200.step import TrainStep
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
gt = scenes.config2(0, n); opt = scenes.perturb(gt, 1)
base_log = np.log(scenes.env_lognormal(128, 256, 2))
cam = ss.fibonacci_cameras(64, 3.5, 800, 800)[5]
env = ss.EnvironmentLight(base_log)
target = ss.render(ss.SurfelCloud(**gt), cam, ss.RenderOptions(), env=env).rgb.contiguous()
cloud = ss.SurfelCloud(**opt)
ts = TrainStep(cloud, env, 800, 800)
ts.gradients([cam], [target])
oenv = O.EnvOracle(base_log)
co = SimpleNamespace(**opt)
ores = O.render(co, cam, env=oenv)
val, g = O.photometric_l1(ores.rgb, target.cpu().numpy())
og = O.backward_image(co, ores, g, None, 0.0, env=oenv)
a = ts.g_env_log.cpu().numpy().astype(np.float64); b = og["env_base_log"]
sc = np.abs(b).max(); err = np.abs(a - b)
bad = err > 1e-3 * np.maximum(np.abs(a), np.abs(b)) + 1e-5 * sc
print("scale", sc, "nbad", bad.sum())
for idx in np.argwhere(bad)[:10]:
    i = tuple(idx); print(i, a[i], b[i], err[i] / sc)
# compare derived-map grads before the adjoint
print("d_diffuse max rel err", np.abs(ts.d_diffuse.cpu().numpy() - og["d_diffuse"]).max() / np.abs(og["d_diffuse"]).max())
print("d_spec max rel err", np.abs(ts.d_spec.cpu().numpy() - og["d_specular"]).max() / np.abs(og["d_specular"]).max())
# env adjoint alone on the oracle's derived-map grads
_, gl = env.env_gradient(og["d_diffuse"], og["d_specular"])
e2 = np.abs(gl.cpu().numpy() - b)
print("adjoint-only nbad", (e2 > 1e-3 * np.abs(b) + 1e-5 * sc).sum(), "max", e2.max() / sc)
