"""Headline benchmark: fwd+bwd views/sec, 1M surfels @ 800^2 (BASELINE config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one inverse-rendering step over 64 views (sharded 64/N per rank),
i.e. per view preprocess+shade, binning/sort, fused forward+L1 loss, backward,
per-surfel chain; then env adjoint, NCCL all-reduce (N>1), Adam, quaternion
renorm and env refresh (paper_2605_05876_b200.step.TrainStep).  Synthetic
seeded data of the config's shape (no dataset ships with the reference):
ground-truth surfels on a noise-displaced unit sphere, targets rendered from
them, optimised parameters = truth + perturbation.  Prints ONE JSON line.

`value` times the step with inputs resident in HBM; `e2e` times the public
TrainStep.step() with the step's target images copied from pinned host memory
every step (overlapped on a copy stream) and the loss read back.  The working
set (56 MB params + 64 x 7.7 MB targets + ~0.3 GB/view of records and pairs)
exceeds the 126 MB L2, so no explicit L2 flush is done between steps.

--impl reference times the CPU oracle (oracle/, the restatement of the
reference's numba/numpy path) on this host's cores for one view of the same
workload (env reduced to 64x128 as BASELINE.md prescribes for config 2).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_SURFELS = 1_000_000
RES = 800
VIEWS_PER_STEP = 64
ENV_SHAPE = (128, 256)
METRIC = "fwd+bwd views/sec, 1M surfels @800², at 1/2/4/8 B200; ncu HBM GB/s vs peak"
UNIT = "views/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_instructions():
    """Executed warp instructions per launch of the rasterisers from the latest
    committed ncu --set full summary (profiles/*_ncu_full.txt): (dict, file)."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_full.txt")))
    if not files:
        return {}, None
    out = {}
    for line in open(files[-1]):
        m = re.match(r"\s*(?:void )?<unnamed>::(\w+).*\| Executed Instructions = ([0-9.]+) inst", line)
        if m and m.group(1) not in out:
            out[m.group(1)] = float(m.group(2))
    return out, os.path.relpath(files[-1], ROOT)


def _traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return None, None
    try:
        with open(files[-1]) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_launch"]), os.path.relpath(files[-1], ROOT)
    except Exception:
        return None, None


def _dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _self_launch(argv, nproc):
    """`bench.py --gpus N` run WITHOUT torchrun: re-exec this script under
    torch.distributed.run with N ranks on this node (one process per GPU,
    rendezvous on 127.0.0.1); rank 0 prints the JSON line.  Returns the
    launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


class _stdout_to_stderr:
    """fd-level redirect of stdout to stderr (C libraries included)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def _check_world(args):
    rank, world, _ = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return rank, world


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo on CPU): every
    rank takes its shard of the step's views, fills a GradPack with
    rank-dependent values, runs the same two-bucket all-reduce TrainStep
    uses, and rank 0 checks the sums and prints one JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2605_05876_b200.step import GradPack, shard_views
    rank, world = _check_world(args)
    if world > 1:
        dist.init_process_group("gloo")
    views = shard_views(VIEWS_PER_STEP, world, rank)
    n, texels = 1000, 32
    pack = GradPack(n, texels, "cpu", dtype=torch.float64)
    pack.flat.copy_(torch.arange(pack.flat.numel(), dtype=torch.float64) * (rank + 1))
    pack.view_count.fill_(float(len(views)))
    work = pack.all_reduce_surfels()
    pack.all_reduce_rest()
    if work is not None:
        work.wait()
    tri = world * (world + 1) / 2
    want = torch.arange(pack.flat.numel(), dtype=torch.float64) * tri
    want[pack.view_count.data_ptr() // 8 - pack.flat.data_ptr() // 8:][:n] = float(VIEWS_PER_STEP)
    ok = bool(torch.equal(pack.flat, want))
    counts = [0] * world
    if world > 1:
        t = torch.zeros(world, dtype=torch.int64)
        t[rank] = len(views)
        dist.all_reduce(t)
        counts = t.tolist()
    else:
        counts = [len(views)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "backend": "gloo" if world > 1 else "none",
                          "views_per_rank": counts, "allreduce_ok": ok}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if not ok:
        raise SystemExit(1)


def _config(extra=None):
    cfg = {"workload": "config2: 1M surfels, 800x800, 64 views/step sharded by view, env 128x256x3, "
                       "L1 loss in linear space, Adam + env refresh per step",
           "surfels": N_SURFELS, "image": [RES, RES], "views_per_step": VIEWS_PER_STEP,
           "env": list(ENV_SHAPE), "cameras": "Fibonacci sphere r=3.5, FOV 45 deg (assumed)",
           "l2": "inputs larger than L2 (no flush)"}
    if extra:
        cfg.update(extra)
    return cfg


# ---------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline)


def cpu_oracle_view(n=N_SURFELS, env_shape=(64, 128), seed=0):
    """One fwd+bwd view of the config-2 workload on the CPU oracle.  Returns
    (seconds, threads, sample description)."""
    from types import SimpleNamespace

    from oracle import oracle as O
    from paper_2605_05876_b200 import scenes
    from paper_2605_05876_b200.camera import fibonacci_cameras

    gt = scenes.config2(seed, n)
    opt = scenes.perturb(gt, seed + 1)
    cam = fibonacci_cameras(VIEWS_PER_STEP, 3.5, RES, RES)[0]
    env = O.EnvOracle(np.log(scenes.env_lognormal(*env_shape, seed + 2)))
    cg, co = SimpleNamespace(**gt), SimpleNamespace(**opt)
    target = O.render(cg, cam, env=env).rgb
    t0 = time.perf_counter()
    res = O.render(co, cam, env=env)
    _, g = O.photometric_l1(res.rgb, target)
    O.backward_image(co, res, g, None, 0.0, env=env)
    dt = time.perf_counter() - t0
    return dt, O.num_threads(), (f"1 view of config 2 ({n} surfels, {RES}x{RES}) fwd+L1+bwd on the C oracle, "
                                 f"env reduced to {env_shape[0]}x{env_shape[1]} (BASELINE.md)")


def env_cpu_timings(shapes=((16, 32), (64, 128)), seed=0):
    """the environment refresh (prefilter) and env_gradient
    (its adjoint) on the CPU oracle at 16x32 and 64x128 (best of 3 / 1)."""
    from oracle import oracle as O
    from paper_2605_05876_b200 import scenes
    out = {}
    for he, we in shapes:
        env = O.EnvOracle(np.log(scenes.env_lognormal(he, we, seed)))
        rng = np.random.default_rng(seed)
        dd, ds = rng.normal(size=(he, we, 3)), rng.normal(size=(env.levels, he, we, 3))
        reps = 3 if he * we <= 4096 else 1
        tr, tg = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            env.refresh()
            tr.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            env.env_gradient(dd, ds)
            tg.append(time.perf_counter() - t0)
        out[f"{he}x{we}"] = {"refresh_ms": 1e3 * min(tr), "env_gradient_ms": 1e3 * min(tg)}
    return out


def env_gpu_timings(shapes=((16, 32), (64, 128), (128, 256), (256, 512)), seed=0):
    """The same two operations on the device (ss_env_refresh / ss_env_adjoint),
    CUDA events, mean of 10 after a warm-up."""
    import torch

    import paper_2605_05876_b200 as ss
    from paper_2605_05876_b200 import scenes
    out = {}
    for he, we in shapes:
        env = ss.EnvironmentLight(np.log(scenes.env_lognormal(he, we, seed)))
        rng = np.random.default_rng(seed)
        dd = torch.tensor(rng.normal(size=(he, we, 3)), device="cuda", dtype=torch.float64)
        ds = torch.tensor(rng.normal(size=(env.levels, he, we, 3)), device="cuda", dtype=torch.float64)
        env.refresh()
        env.env_gradient(dd, ds)
        res = {}
        for name, fn in (("refresh_ms", env.refresh), ("env_gradient_ms", lambda: env.env_gradient(dd, ds))):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                fn()
            b.record()
            b.synchronize()
            res[name] = a.elapsed_time(b) / 10
        out[f"{he}x{we}"] = res
    return out


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    for _ in range(max(args.warmup, 0) and 1):
        cpu_oracle_view(n=100_000)
    times = []
    for _ in range(args.steps):
        dt, cores, sample = cpu_oracle_view()
        times.append(dt)
    v = 1.0 / float(np.mean(times))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
            "data": "synthetic", "config": _config({"sample": sample}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------
# the other BASELINE configs (configs[0, 1, 3] and the one-GPU slice of 4):
# views/s of the same training step on their scenes, resident inputs


def _config_workload(cfg):
    """(gt, init, env_base, cameras, W, H, extra) of BASELINE config `cfg`."""
    import paper_2605_05876_b200 as ss
    from paper_2605_05876_b200 import scenes
    if cfg == 0:
        gt = scenes.config0(0, 10_000)
        init = dict(gt)
        init["centers"] = (gt["centers"] + np.random.default_rng(1).normal(0, 0.01, gt["centers"].shape)).astype(
            np.float32)
        cams = [ss.Camera.perspective(128, 128, 40.0, (3.0, 0.0, 0.0), (0.0, 0.0, 0.0))]
        return gt, init, scenes.env_lognormal(16, 32, 2), cams, 128, 128, {}
    if cfg == 1:
        gt = scenes.config1(0, 200_000)
        return gt, scenes.perturb(gt, 1), scenes.env_lognormal(64, 128, 2), ss.fibonacci_cameras(8, 3.5, 512, 512), \
            512, 512, {}
    if cfg == 3:
        gt = scenes.config3(0, 500_000)
        return gt, scenes.perturb(gt, 1), scenes.env_lognormal(64, 128, 2), \
            ss.fibonacci_cameras(16, 3.5, 1024, 1024), 1024, 1024, {}
    if cfg == 4:
        gt = scenes.config2(0, 4_000_000, amp=0.12, octaves=5)
        cams = ss.fibonacci_cameras(128, 3.5, 1920, 1080)[:16]  # one GPU's 16 of the step's 128 views
        return gt, scenes.perturb(gt, 1), scenes.env_lognormal(256, 512, 2), cams, 1920, 1080, \
            {"max_surfels": 4_200_000, "quantile": 0.95}
    raise ValueError(cfg)


def run_config(cfg, steps=None, warmup=3):
    """views/s of the training step (L1, Adam, env refresh) on config `cfg`;
    config 4 adds the per-step refinement pass (q = 0.95, budget 1.05 N) and
    the neighbour-index rebuild, timed separately and inside the step."""
    import torch

    import paper_2605_05876_b200 as ss
    from paper_2605_05876_b200.densify import DensifyStats
    from paper_2605_05876_b200.step import TrainStep
    gt, init, env_base, cams, W, H, extra = _config_workload(cfg)
    steps = steps or {0: 50, 1: 20}.get(cfg, 3)
    gt_env = ss.EnvironmentLight.from_base(env_base)
    gtc = ss.SurfelCloud(**gt)
    targets = [ss.render(gtc, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
    del gtc
    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight(np.log(env_base))
    refine = "max_surfels" in extra
    ts = TrainStep(cloud, env, W, H, streams=3, surfel_capacity=extra.get("max_surfels"))
    ts.size_pairs(cams[:2])
    index = ss.NeighborIndex(ts.cloud, k=8) if refine else None
    ev = lambda: torch.cuda.Event(enable_timing=True)
    ref_ms, knn_ms, sizes = [], [], []

    graph = [not refine]  # CUDA-graph replay of the gradient pass (the refining step rebinds the cloud)

    def one():
        ts.step(cams, targets, graph=graph[0])
        if refine:
            stats = DensifyStats.zeros(len(ts.cloud))
            stats.accumulate(ts.grads["ss_grad"], ts.view_count)
            a, b, c = ev(), ev(), ev()
            a.record()
            ts.refine(stats, index.mean_dist, extra["max_surfels"], quantile=extra["quantile"])
            b.record()
            index.rebuild(ts.cloud)
            c.record()
            return a, b, c
        return None

    def timed():
        for _ in range(warmup):
            one()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        marks = [one() for _ in range(steps)]
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps, marks

    ms, marks = timed()
    out = {"views_per_s": len(cams) / (ms / 1e3), "ms_per_step": ms, "views_per_step": len(cams),
           "surfels": len(init["centers"]), "image": [W, H], "env": list(env_base.shape[:2]),
           "cuda_graph": graph[0]}
    if graph[0]:  # the same step issued eagerly (Python + ctypes launches per view)
        graph[0] = False
        ms_e, _ = timed()
        out["views_per_s_eager"] = len(cams) / (ms_e / 1e3)
    if refine:
        ref_ms = [a.elapsed_time(b) for a, b, _ in marks]
        knn_ms = [b.elapsed_time(c) for _, b, c in marks]
        out.update({"refinement_ms": float(np.mean(ref_ms)), "knn_rebuild_ms": float(np.mean(knn_ms)),
                    "surfels_after": len(ts.cloud), "quantile": extra["quantile"],
                    "max_surfels": extra["max_surfels"],
                    "step": "16 of the 128 views of a step (the per-GPU slice at 8 GPUs): fwd+bwd, env adjoint, "
                            "Adam, env refresh, then refine_topology (device) and the KNN rebuild"})
    del ts
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2605_05876_b200 as ss
    from paper_2605_05876_b200 import scenes
    from paper_2605_05876_b200.step import TrainStep

    rank, world = _check_world(args)
    local = _dist_env()[2]
    torch.cuda.set_device(local)
    # SS_COLLECTIVES=force under torchrun with one rank: the NCCL path (process
    # group, all-reduces, max-over-ranks timing) on a single GPU (self-test)
    multi = world > 1 or (os.environ.get("SS_COLLECTIVES") == "force" and "WORLD_SIZE" in os.environ)
    if multi:
        # NCCL prints its version line on stdout at communicator creation
        # (NCCL_DEBUG=VERSION in this image): create it with fd 1 on stderr,
        # so stdout carries only the JSON line
        with _stdout_to_stderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
    from paper_2605_05876_b200.step import shard_views
    my_views = shard_views(VIEWS_PER_STEP, world, rank)

    gt = scenes.config2(0, N_SURFELS)
    init = scenes.perturb(gt, 1)
    env_base = scenes.env_lognormal(*ENV_SHAPE, 2)
    cams_all = ss.fibonacci_cameras(VIEWS_PER_STEP, 3.5, RES, RES)
    cams = [cams_all[i] for i in my_views]

    # targets rendered from ground truth (linear HDR), then kept resident
    gt_cloud = ss.SurfelCloud(**gt)
    gt_env = ss.EnvironmentLight.from_base(env_base)
    targets = [ss.render(gt_cloud, c, ss.RenderOptions(), env=gt_env).rgb.contiguous() for c in cams]
    del gt_cloud
    torch.cuda.synchronize()

    cloud = ss.SurfelCloud(**init)
    env = ss.EnvironmentLight(np.log(env_base) + np.random.default_rng(3).normal(0, 0.1, env_base.shape))
    ts = TrainStep(cloud, env, RES, RES, streams=int(os.environ.get("SS_STREAMS", "3")))
    ts.size_pairs(cams[:4])
    stream = torch.cuda.current_stream()

    def one_step():
        return ts.step(cams, targets)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if ts.check_overflow():
        ts.size_pairs(cams, slack=1.3)
        one_step()

    # ---- timed region: inputs resident in HBM ----
    clocks = Clocks(local) if rank == 0 else None
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the timed steps carry no instrumentation (per-kernel events between the
    # launches cost ~3% of the step by perturbing the worker streams' overlap)
    ev0.record(stream)
    for _ in range(args.steps):
        one_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    step_ms = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop() if clocks else None
    # one more step with events around every stage launch (the in-step
    # per-kernel times: concurrent streams, so each span includes overlap)
    ts.kernel_events = []
    one_step()
    torch.cuda.synchronize()
    kev = ts.kernel_events
    ts.kernel_events = None
    t = torch.tensor([step_ms], device="cuda", dtype=torch.float64)
    if multi:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms = float(t.item())
    value = VIEWS_PER_STEP / (step_ms / 1e3)

    # dominant kernel (raster backward) share and roofline, live CUDA events
    per_kernel = {}
    for name, a, b in kev:
        per_kernel.setdefault(name, []).append(a.elapsed_time(b))
    ts.collect_stats = True
    one_step()
    ts.collect_stats = False
    stats = ts.last_stats()
    # the same kernels with the views serialised on one worker stream: their
    # own launch durations (in the timed region the worker streams overlap,
    # so each event pair also spans the other streams' concurrent kernels)
    ts.active_streams, ts.kernel_events = 1, []
    one_step()
    torch.cuda.synchronize()
    iso = {}
    for name, a, b in ts.kernel_events:
        iso.setdefault(name, []).append(a.elapsed_time(b))
    ts.active_streams, ts.kernel_events = None, None
    # per-step fixed stages, timed on their own: they are inside
    # every timed step above as well
    fixed = ts.fixed_costs()
    fixed["env_by_size"] = env_gpu_timings()  # BASELINE.md §2 sizes (+ configs 2 and 4)
    if world == 1:
        # the density-aware refinement scan on this step's statistics, on the
        # device (refine_topology: isolation, prune, quantile, budget, split,
        # Adam remap), and the KNN rebuild the reference runs after it
        from paper_2605_05876_b200.densify import DensifyStats, refine_topology
        st = DensifyStats.zeros(len(cloud))
        st.accumulate(ts.grads["ss_grad"], ts.view_count)
        knn = ss.NeighborIndex(cloud, k=8)
        refine_topology(cloud, st, knn.mean_dist, max_surfels=int(1.05 * len(cloud)))  # warm-up
        ra, rb, rc = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        ra.record(stream)
        _, imap, reasons = refine_topology(cloud, st, knn.mean_dist, max_surfels=int(1.05 * len(cloud)))
        rb.record(stream)
        knn.rebuild(cloud)
        rc.record(stream)
        torch.cuda.synchronize()
        fixed["refinement_scan"] = ra.elapsed_time(rb)
        fixed["knn_rebuild"] = rb.elapsed_time(rc)
        fixed["refinement_result"] = {"surfels_out": int(imap.numel()),
                                      **{k: int(v) for k, v in reasons.items() if np.isscalar(v)}}
        del imap

    # ---- e2e: public API with host-resident targets ----
    host_targets = [tg.cpu().pin_memory() for tg in targets]
    for _ in range(2):
        ts.step_host(cams, host_targets).item()
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    e0 = time.perf_counter()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(args.steps):
        ts.step_host(cams, host_targets).item()
    eb.record(stream)
    torch.cuda.synchronize()
    e_ms = ea.elapsed_time(eb) / args.steps
    et = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
    if multi:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e_ms = float(et.item())
    h2d = sum(h.numel() * h.element_size() for h in host_targets) * world
    e2e = {"value": VIEWS_PER_STEP / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": 4 * world, "wall_ms_per_step": 1e3 * (time.perf_counter() - e0) / args.steps}

    # ---- the reference fit loss: hdr-loss tone map +
    # 0.8 L1 + 0.2 (1 - SSIM) on the device, deferred-loss kernels ----
    launches = ts.launches_per_step * args.steps
    last_loss = float(ts.loss_f.item())
    del ts
    torch.cuda.empty_cache()
    tp = TrainStep(cloud, env, RES, RES, streams=int(os.environ.get("SS_STREAMS", "3")), loss="photometric")
    tp.size_pairs(cams[:4])
    for _ in range(2):
        tp.step(cams, targets)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pa.record(stream)
    for _ in range(args.steps):
        tp.step(cams, targets)
    pb.record(stream)
    torch.cuda.synchronize()
    p_ms = pa.elapsed_time(pb) / args.steps
    pt = torch.tensor([p_ms], device="cuda", dtype=torch.float64)
    if multi:
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    photometric = {"value": VIEWS_PER_STEP / (float(pt.item()) / 1e3), "unit": UNIT,
                   "loss": "tone_map hdr-loss, 0.8 L1 + 0.2 (1 - SSIM 11x11) (train.py:194-199)",
                   "ms_per_step": float(pt.item())}
    # the main-phase fit loss: + depth consolidation, cons_scale =
    # lambda_cons / (extent * npix) with the reference defaults (lambda_cons
    # 100, train.py:44, 208-210) and extent 1 (the unit-sphere scene)
    tp.cons_scale = 100.0 / (1.0 * RES * RES)
    for _ in range(2):
        tp.step(cams, targets)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    pa.record(stream)
    for _ in range(args.steps):
        tp.step(cams, targets)
    pb.record(stream)
    torch.cuda.synchronize()
    pt = torch.tensor([pa.elapsed_time(pb) / args.steps], device="cuda", dtype=torch.float64)
    if multi:
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    photometric_cons = {"value": VIEWS_PER_STEP / (float(pt.item()) / 1e3), "unit": UNIT,
                        "loss": "the above + depth consolidation, cons_scale = 100 / (1 * 800 * 800) "
                                "(train.py:208-213)", "ms_per_step": float(pt.item())}
    del tp

    if rank != 0:
        if multi:
            dist.destroy_process_group()
        return

    configs = {}
    if world == 1 and not args.no_configs:
        for c in (0, 1, 3, 4):
            try:
                configs[f"config{c}"] = run_config(c)
            except Exception as e:  # reported, never fatal for the headline
                configs[f"config{c}"] = {"error": repr(e)[:200]}
    peak, peak_kind = _peaks()
    traffic, traffic_src = _traffic()
    P, Nk = stats["pairs_mean"], stats["kept_mean"]
    HW = RES * RES
    bwd_ms = float(np.mean(iso.get("train_backward", [float("nan")])))
    bwd_ms_step = float(np.mean(per_kernel.get("train_backward", [float("nan")])))
    # algorithmic (compulsory) bytes per launch of the record-parallel
    # backward: every kept record read once (96 B) and its 80 B accumulator
    # row written, the per-pixel layer header read once (32 B/px) and the
    # 16 B coefficient texel of every (pixel, layer) once (LP = sum over
    # pixels of the layer count, measured on the step's views)
    LP = stats.get("layer_pixels_mean", 0.0)
    bwd_bytes = 96.0 * Nk + 80.0 * Nk + 32.0 * HW + 16.0 * LP
    achieved = bwd_bytes / (bwd_ms / 1e3) / 1e9
    view_bytes = 176.0 * N_SURFELS + 352.0 * Nk + 236.0 * P + 40.0 * HW
    # issue-slot roofline of the two rasterisers (issue-bound: nothing on the
    # path is a contraction, so the SM's instruction issue rate -- 4 warp
    # instructions per clock per SM -- is their ceiling, not HBM)
    instr, instr_src = _ncu_instructions()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    issue_peak = sms * 4 * mhz * 1e6
    issue = {"unit": "warp instructions/s", "peak": issue_peak,
             "peak_basis": f"{sms} SMs x 4 issue slots x {mhz:.0f} MHz (median SM clock under load)",
             "instructions_source": instr_src, "kernels": {}}
    for name, kern, ms in (("train_forward", ("raster_fwd_kernel",), iso.get("train_forward")),
                           ("train_backward", ("splat_bwd_kernel", "big_bwd_kernel"), iso.get("train_backward"))):
        n_instr = sum(instr.get(k, 0.0) for k in kern)
        if n_instr and ms:
            t = float(np.mean(ms)) / 1e3
            issue["kernels"][name] = {"warp_instructions_per_launch": n_instr, "launch_ms": t * 1e3,
                                      "achieved": n_instr / t, "frac": n_instr / t / issue_peak,
                                      "ncu_kernels": list(kern)}
    cpu = None
    if world == 1 and not args.no_cpu:
        dt, cores, sample = cpu_oracle_view()
        cpu = {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "env": env_cpu_timings()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config({"parallelism": f"dp{world} over views", "pairs_per_view": P, "kept_per_view": Nk,
                                 "layer_pixels_per_view": LP,
                                 "collective": (f"NCCL all-reduce, {dist.get_world_size()} rank(s), 2 buckets per step"
                                                if multi else "none (one process)")}),
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "kernel": "record backward (ss_train_backward_records: area classes, splat_bwd, big rects)",
                     "algorithmic_bytes_per_launch": bwd_bytes,
                     "algorithmic_bytes_formula": "96 Nk + 80 Nk + 32 HW + 16 LP (records, accumulator rows, "
                                                  "pixel headers, (pixel, layer) coefficients)",
                     "avg_launch_ms": bwd_ms,
                     "avg_launch_ms_in_step": bwd_ms_step,
                     "timing": "CUDA events around each ss_train_backward_records call on its worker stream, one "
                               "step with the views serialised (avg_launch_ms); in the timed 3-stream step the "
                               "same events also span the other streams' kernels (avg_launch_ms_in_step)",
                     "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json)"},
        "issue_roofline": issue,
        "view_roofline": {"bytes_per_view": view_bytes,
                          "achieved_gbs": view_bytes * VIEWS_PER_STEP / world / (step_ms / 1e3) / 1e9,
                          "frac": view_bytes * VIEWS_PER_STEP / world / (step_ms / 1e3) / 1e9 / peak},
        "kernel_ms": {k: float(np.mean(v)) for k, v in iso.items()},
        "kernel_ms_in_step": {k: float(np.mean(v)) for k, v in per_kernel.items()},
        "per_step_fixed_ms": fixed,
        "photometric_loss_step": photometric,
        "photometric_cons_loss_step": photometric_cons,
        "other_configs": configs,
        "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
        "loss": last_loss,
    }
    print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs 0/1/3/4 lines")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing on CPU (gloo), no GPU work")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(sys.argv[1:], args.gpus))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
