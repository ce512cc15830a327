"""Helper of tests/test_gpu_nccl.py (run under torch.distributed.run with ONE
rank and SS_COLLECTIVES=force): the TrainStep gradient pass through the NCCL
process group -- async per-surfel bucket on NCCL's stream, then the env /
loss / status bucket -- against the same pass without collectives.  One rank
makes the all-reduce an identity, so the packs must agree up to the float
atomics' summation order (derived-map texels, big records); what
this checks on a single GPU is the NCCL plumbing (communicator bound to the
device, async work handle, stream ordering against the worker streams)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_05876_b200 as ss  # noqa: E402
from paper_2605_05876_b200 import scenes  # noqa: E402
from paper_2605_05876_b200.step import TrainStep, collectives_on  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
assert dist.get_backend() == "nccl" and os.environ.get("SS_COLLECTIVES") == "force"

gt = scenes.config0(0, 3000)
init = scenes.perturb(gt, 1)
env_base = scenes.env_lognormal(16, 32, 2)
cams = ss.fibonacci_cameras(4, 3.0, 96, 96, fov_y_deg=40.0)
gt_env = ss.EnvironmentLight.from_base(env_base)
gtc = ss.SurfelCloud(**gt)
targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]


def packed(force):
    os.environ["SS_COLLECTIVES"] = "force" if force else "off"
    assert collectives_on() == force
    ts = TrainStep(ss.SurfelCloud(**init), ss.EnvironmentLight(np.log(env_base)), 96, 96, streams=1)
    ts.size_pairs(cams[:2])
    ts.gradients(cams, targets)
    if force:  # the per-surfel bucket really goes through NCCL (a work handle)
        work = ts.pack.all_reduce_surfels()
        assert work is not None
        work.wait()
    torch.cuda.synchronize()
    return ts.pack.flat.clone()


a = packed(True)
b = packed(False)
assert torch.isfinite(a).all() and a.abs().sum() > 0
# one rank: identity up to the order of float atomics (max |a-b| ~1e-10 of O(1) entries)
scale = float(b.abs().max())
assert torch.allclose(a, b, rtol=1e-6, atol=1e-9 * scale), float((a - b).abs().max())
dist.destroy_process_group()
print("NCCL_SELFTEST_OK", a.numel())
