"""Benchmark of the hot path (BASELINE.json metric: render FPS / train it/s on B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4]
    python bench.py --impl reference ...      (the reference's CPU implementation)

Default workload at N=1: BASELINE config 4, the largest single-GPU config -- one step =
forward render of N=6M SH-3 Gaussians at 3840x2160 + 0.8 L1 + 0.2 D-SSIM against the seed-1
target set's render + the full backward, all on the device through libbsr.so; config 1
(100k, 800x800, + Adam) is measured after it and nested under "secondary".  At N>1 the
default is config 3: the 32-view batch (3M Gaussians, 1600x1067) split 32/N across ranks
(one process per GPU, NCCL all-reduce of the flat gradient buffer, then Adam; strong
scaling).  `--gpus N` without a torchrun environment relaunches itself under
torch.distributed.run with N local ranks.  --config c1|c2|c3|c4 picks a workload.

Timing: W warm-up steps, then K steps of the captured step graph, each timed with CUDA
events on the launching stream (L2 flushed with a 256 MiB write between steps, outside the
events), bracketed by barrier + synchronize, max over ranks.  Stage times / pair counts for
the roofline come from libbsr's caller-owned events and device counters (eager steps before
the timed region).  e2e: the same step through the public API (render_tiled,
training.loss_into, render_backward, adam_step) with every step's inputs copied from
pinned host memory and its loss read back, copies inside the timing.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FP32_FLOP_PER_PAIR_FWD = 27  # SURVEY 8(d), counted from _raster.pyx:107-123
FP32_FLOP_PER_PAIR_BWD = 80  # SURVEY 8(d), counted from _raster.pyx:197-241
SM_COUNT = 148
FP32_LANES_PER_SM = 128


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm_gbs=float(p["hbm_gbs"]), sm_max_mhz=float(p.get("sm_max_mhz", 1965.0)),
                    source="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback (B200_PROFILING.md)")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML on a background
    thread every ~10 ms (nvidia-smi -lms cannot resolve sub-second regions)."""

    # nvmlClocksEventReasons bits (nvml.h)
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index=0, period_s=0.01):
        self.gpu, self.period = gpu_index, period_s
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.thread, self.stop_flag = None, False

    def _run(self, nv, h):
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                try:
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for b, nm in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._run, args=(nv, h), daemon=True)
            self.thread.start()
        except Exception as e:
            self.error = repr(e)

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {getattr(self, 'error', '')}"]}
        self.stop_flag = True
        self.thread.join(timeout=2)
        sm = self.samples
        loaded = [v for v in sm if v >= 0.5 * (self.max_mhz or max(sm))] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz, "samples": len(sm),
                "reasons": sorted(self.reasons), "source": "NVML, ~10 ms period, during the timed region"}


# ----------------------------------------------------------------------------- distributed
def dist_setup(n_gpus):
    """torch.distributed from the torchrun environment: NCCL, one GPU per rank.
    BSR_DIST_BACKEND=gloo runs the same multi-rank code path over gloo (several ranks may
    then share one GPU: a functional check of the launcher, the sharded exchange and the
    JSON line on a one-GPU box; not a performance configuration)."""
    from paper_2501_18630_b200 import distributed as dd

    if int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return dd.init(None)
    backend = os.environ.get("BSR_DIST_BACKEND", "nccl")
    # the communicator's init lines (ranks, transports, NVLS) on stderr, also when the
    # driver's torchrun launched the ranks instead of spawn_ranks
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if backend == "gloo":
        import torch

        torch.cuda.set_device(0 if torch.cuda.device_count() == 1 else int(os.environ.get("LOCAL_RANK", "0")))
        return dd.init("gloo")
    return dd.init(backend)


def barrier(world):
    import torch

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x, world):
    from paper_2501_18630_b200 import distributed as dd

    return dd.max_over_ranks(x) if world > 1 else float(x)


def sum_over_ranks(x, world):
    from paper_2501_18630_b200 import distributed as dd

    return dd.sum_over_ranks(x) if world > 1 else float(x)


# ----------------------------------------------------------------------------- workloads
def rank_cameras(cfg, rank, world, views_per_gpu):
    """Cameras of this rank.  c1: view r of a y-orbit at radius 4 (rank 0 == config-1
    camera); c3: contiguous share of the 32 config-3 cameras."""
    from paper_2501_18630_b200.distributed import orbit_cameras, partition_views
    from paper_2501_18630_b200.scenes import make_workload

    if cfg == "c1":
        cams = orbit_cameras(world * views_per_gpu)
        return [cams[k] for k in partition_views(len(cams), world, rank)]
    # the hemisphere cameras come from their own stream (scenes.camera_rng): the same views
    # as the full-size workload that cpu_reference_step_fn renders
    if cfg == "c3":
        wl_cams = make_workload("c3", seed=0, n=16).cameras
        return [wl_cams[k] for k in partition_views(len(wl_cams), world, rank)]
    return make_workload(cfg, seed=0, n=16).cameras


def build_b200(cfg, rank, world, views_per_gpu):
    import torch

    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.scenes import make_workload, target_scene
    from paper_2501_18630_b200.training import TrainStep, render_targets

    n = {"c1": 100_000, "c2": 1_000_000, "c3": 3_000_000, "c4": 6_000_000}[cfg]
    wl = make_workload(cfg, seed=0, n=n, views=1 if cfg != "c3" else 32)
    prims = PrimitiveSet.from_scene(wl.scene)
    cams = rank_cameras(cfg, rank, world, views_per_gpu)
    bg = wl.background
    if cfg == "c2":
        return dict(kind="render", prims=prims, cams=cams, bg=bg, scene=wl.scene, world=world)
    tgt = PrimitiveSet.from_scene(target_scene(cfg, 1, n))
    targets = render_targets(tgt, cams, bg)
    del tgt
    torch.cuda.empty_cache()
    pg = None
    if world > 1:
        import torch.distributed as dist

        pg = dist.group.WORLD
    step = TrainStep(prims, cams, targets, bg, process_group=pg)
    return dict(kind="train", prims=prims, cams=cams, bg=bg, step=step, targets=targets, scene=wl.scene,
                adam=(cfg != "c4"), world=world)


def run_step(w, prof=None):
    """One hot-path step; returns the number of views processed."""
    import torch

    if "graph" in w:  # captured CUDA graph of the whole step (see make_graph)
        w["graph"].replay()
        return len(w["cams"])

    from paper_2501_18630_b200.rasterizer import _prims_scene_c, forward_raw, outputs_c

    if w["kind"] == "render":
        if "color" not in w:
            c = w["cams"][0]
            w["color"] = torch.empty((c.height, c.width, 3), dtype=torch.float32, device="cuda")
            w["frame"] = None
            w["sc"] = _prims_scene_c(w["prims"])
        for i, cam in enumerate(w["cams"]):
            w["frame"] = forward_raw(w["sc"], cam, w["bg"], outputs_c(color=w["color"]), frame=w["frame"],
                                     check=False, profile=None if prof is None else prof.fwd(i))
        return len(w["cams"])
    st = w["step"]
    st.profile = prof
    st.step(check=False, adam=w["adam"])
    return len(w["cams"])


def capture_mode(w):
    """Multi-rank steps capture the NCCL all-reduce: thread-local capture mode keeps the
    process group's watchdog thread (event queries) from invalidating the capture."""
    return "thread_local" if w.get("world", 1) > 1 else "global"


def make_graph(w, prof=None, warmup=2):
    """Capture one whole step (all views, all kernels, all-reduce, Adam) in a CUDA graph."""
    import torch

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warmup):
            run_step(w, prof)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode=capture_mode(w)):
        run_step(w, prof)
    torch.cuda.synchronize()
    w["graph"] = g


def flush_l2(buf):
    buf.zero_()


def timed_loop(w, steps, world, prof=None, l2=None):
    """K device-timed steps (CUDA events on the launching stream; L2 flush outside)."""
    import torch

    total_ms, views = 0.0, 0
    barrier(world)
    for _ in range(steps):
        if l2 is not None:
            flush_l2(l2)
        if prof is not None and "graph" not in w:
            # profiled eager steps: a ~10 ms spin kernel lets the host enqueue the whole step
            # before the GPU reaches it, so stage events measure device time, not launch gaps
            torch.cuda._sleep(20_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        views += run_step(w, prof)
        e.record()
        e.synchronize()
        total_ms += s.elapsed_time(e)
        if prof is not None:
            prof.collect_step(w)
    barrier(world)
    return total_ms, views


def e2e_loop(w, steps, world):
    """The step captured in CUDA graphs together with its per-step host inputs (pinned) and
    the result read back, copies inside the timing (reported as extra.e2e_graph; the
    headline e2e is e2e_api_loop).

    Every step copies its inputs host->device (the per-view target images; config 2 has
    none) and reads its result device->host (the loss values; the rendered image for
    config 2).  The step and its copies are captured together into two CUDA graphs
    (alternating staging buffers), the way a training / serving loop would pipeline them:
    graph i uploads step i+1's inputs into the other staging buffer on a forked copy
    branch while step i reads its own, config 2 downloads frame i-1 while frame i
    renders; the host reads step i-1's result before launching step i+1."""
    import torch

    main, cs = torch.cuda.current_stream(), torch.cuda.Stream()
    train = w["kind"] == "train"
    step_graph = w.pop("graph", None)  # the step is captured again inside the e2e graphs
    if train:
        # page-locked buffers from the pinned allocator: Tensor.pin_memory() moved only
        # ~11 GB/s host->device on the B200 box, torch.empty(pin_memory=True) ~54 GB/s
        # (scripts/h2d_probe.py)
        # (scripts/h2d_probe.py); fresh page-locked buffers also move slowly for their first
        # few hundred copies on this box (scripts/e2e_probe4.py), so they are created once per
        # workload and exercised before the timed region
        if "e2e_host" not in w:
            w["e2e_host"] = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t.cpu())
                             for t in w["targets"]]
        host = w["e2e_host"]
        stage = [[torch.empty_like(t) for t in w["targets"]] for _ in range(2)]
        res_dev = w["step"].loss_values
        bi = sum(h.numel() * h.element_size() for h in host)
    else:
        if "color" not in w:
            run_step(w)
        res_dev = w["color"]
        stage = [torch.empty_like(res_dev) for _ in range(2)]
        bi = 0
    res_host = [torch.empty(res_dev.shape, dtype=res_dev.dtype, pin_memory=True) for _ in range(2)]
    bo = res_dev.numel() * res_dev.element_size()

    graphs = []
    for b in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode=capture_mode(w)):
            cur = torch.cuda.current_stream()
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                if train:  # next step's inputs
                    for dst, h in zip(stage[b ^ 1], host):
                        dst.copy_(h, non_blocking=True)
                else:  # previous frame's image
                    res_host[b ^ 1].copy_(stage[b ^ 1], non_blocking=True)
            if train:
                # graph b's step reads its targets straight from staging buffer b (no D2D copy)
                w["step"].targets = list(stage[b])
                run_step(w)
                res_host[b].copy_(res_dev, non_blocking=True)  # the step's loss values
            else:
                run_step(w)
                stage[b].copy_(res_dev, non_blocking=True)
            cur.wait_stream(cs)
        graphs.append(g)
    if train:
        w["step"].targets = list(w["targets"])
    for _ in range(10):  # first launches upload the graphs
        for g in graphs:
            g.replay()
    torch.cuda.synchronize()
    warm_host_link()  # steady-state host link (scripts/h2d_probe.py)

    done = [torch.cuda.Event(), torch.cuda.Event()]
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(main)
    views = 0
    if train:  # first step's inputs
        for dst, h in zip(stage[0], host):
            dst.copy_(h, non_blocking=True)
    for i in range(steps):
        graphs[i % 2].replay()
        done[i % 2].record(main)
        views += len(w["cams"])
        if i >= 1:
            done[(i - 1) % 2].synchronize()  # the host has step i-1's result
    if not train:  # last frame's image
        res_host[(steps - 1) % 2].copy_(stage[(steps - 1) % 2], non_blocking=True)
    e.record(main)
    e.synchronize()
    ms = s.elapsed_time(e)
    barrier(world)
    if step_graph is not None:
        w["graph"] = step_graph
    return ms, views, bi, bo


class BenchProfiler:
    """Per-view stage times + pair counts from libbsr's profiling hooks (bsr_profile)."""

    def __init__(self, n_views):
        from paper_2501_18630_b200.rasterizer import StageProfiler

        self.sp = StageProfiler(n_views)

    def mark_loss(self, i, end=False):
        self.sp.mark_loss(i, end)

    def mark_adam(self, end=False):
        self.sp.mark_adam(end)

    def mark_color(self, end=False):
        self.sp.mark_color(end)

    def fwd(self, i):
        return self.sp.fwd(i)

    def bwd(self, i):
        return self.sp.bwd(i)

    def collect_step(self, w):
        self.sp.collect_step()


def kernel_launches_per_step(w):
    from paper_2501_18630_b200.rasterizer import frame_status

    cam = w["cams"][0]
    # pre (+ tile counts), bin scan, bin scatter, per-tile sort, raster, replay
    fwd = 1 + 1 + 1 + 1 + 1 + 1
    if w["kind"] == "render":
        return fwd * len(w["cams"])
    per_view = fwd + 2 + 5  # + loss (maps, grad+finish) + backward (zero, raster, replay, chain, fp64 geometry chain)
    st = w.get("step")
    color = 1 if st is not None and getattr(st, "drgb", None) is not None else 0  # deferred colour chain
    return per_view * len(w["cams"]) + color + (1 if w["adam"] else 0)  # Adam (fused step bump)


# ----------------------------------------------------------------------------- CPU baseline
def cpu_reference_step_fn(cfg, threads):
    """One step of the reference's CPU implementation: the reference's own compiled raster
    core (oracle/_ref, built from /root/reference by oracle/Makefile) driven by the oracle's
    numpy restatement of the per-frame glue (projection, SH adapter, sort, binning, chain),
    L1 + D-SSIM and Adam.  Returns (step_fn, description)."""
    from oracle import pipeline as orc
    from paper_2501_18630_b200.scenes import make_workload, target_scene

    kind = "reference" if orc.have_ref_core() else "port"
    core = "ref" if kind == "reference" else "c"
    n = {"c1": 100_000, "c2": 1_000_000, "c3": 3_000_000, "c4": 6_000_000}[cfg]
    wl = make_workload(cfg, seed=0, n=n, views=1 if cfg != "c3" else 32)
    scene = wl.scene.astype(np.float64)
    cam = rank_cameras(cfg, 0, 1, 1)[0] if cfg in ("c1",) else wl.cameras[0]
    bg = wl.background
    if cfg == "c2":
        def step():
            orc.forward(scene, cam, bg, core=core, threads=threads)
        return step, kind, f"{cfg}: one forward render on {threads} host threads"
    tgt = orc.forward(target_scene(cfg, 1, n).astype(np.float64), cam, bg, core=core, threads=threads)["color"]
    params = {k: v.copy() for k, v in scene.arrays().items() if k != "shapes"}
    m = {k: np.zeros_like(v) for k, v in params.items()}
    v2 = {k: np.zeros_like(v) for k, v in params.items()}
    lrs = {k: (1.6e-4 if k == "positions" else 5e-3) for k in params}
    state = {"t": 0}

    def step():
        fwd = orc.forward(scene, cam, bg, core=core, threads=threads)
        _, d_img = orc.loss(fwd["color"], tgt)
        g = orc.backward(scene, cam, bg, d_img, fwd, core=core, threads=threads)
        if cfg != "c4":
            state["t"] += 1
            orc.adam_step(params, {k: g[k] for k in params}, m, v2, state["t"], lrs)
    desc = (f"{cfg}: one training view (fwd + L1/D-SSIM + bwd" + (" + Adam" if cfg != "c4" else "") +
            f") on {threads} host threads")
    if cfg == "c3":
        desc += "; 1 of the 32 views per step (multiply ms by 32 for one iteration)"
    return step, kind, desc


def cpu_baseline(cfg, budget_s=15.0):
    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    step, kind, desc = cpu_reference_step_fn(cfg, threads)
    if cfg in ("c1", "c2"):
        step()  # warm-up (first-touch, BLAS init); configs 3 / 4 take 10-40 s per step: one timed step
    t0 = time.perf_counter()
    k = 0
    while True:
        step()
        k += 1
        if time.perf_counter() - t0 >= budget_s or k >= 10:
            break
    dt = (time.perf_counter() - t0) / k
    return dict(value=1.0 / dt, unit=unit_for(cfg), cores=threads, kind=kind,
                sample=f"{desc}; {k} steps, {dt * 1e3:.0f} ms/step", ms_per_step=dt * 1e3)


def unit_for(cfg):
    return {"c1": "views/s", "c2": "frames/s", "c3": "views/s", "c4": "it/s"}[cfg]


def metric_for(cfg):
    return {
        "c1": "train it/s (config 1: fwd + 0.8 L1 + 0.2 D-SSIM + bwd + Adam, N=100k SH-3, 800x800)",
        "c2": "render FPS (config 2: forward, N=1M SH-3, 1920x1080)",
        "c3": "train views/s (config 3: 32-view batch fwd + loss + bwd, all-reduce, Adam; N=3M SH-3, 1600x1067)",
        "c4": "fwd+bwd it/s (config 4: N=6M SH-3, 3840x2160, L1 + D-SSIM upstream)",
    }[cfg]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    step, kind, desc = cpu_reference_step_fn(args.config, threads)
    warm = min(args.warmup, 1) if args.config in ("c1", "c2", "c3") else 0
    steps = max(1, min(args.steps, 5 if args.config in ("c1", "c2") else 1))
    for _ in range(warm):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    views = 1
    val = views / dt
    line = {
        "impl": "reference", "metric": metric_for(args.config), "value": val, "unit": unit_for(args.config),
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config generators)",
        "config": {"workload": args.config},
        "cpu_baseline": {"value": val, "unit": unit_for(args.config), "cores": threads, "kind": kind,
                         "sample": f"{desc}; steps capped at {steps} to bound the run"},
        "e2e": {"value": val, "unit": unit_for(args.config), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- e2e (public API)
def e2e_api_loop(w, steps, world):
    """The same step through the package's public API -- render_tiled, training.loss_into,
    render_backward (+ all-reduce + adam_step for the training configs) -- eagerly, with
    every step's inputs copied host->device from pinned memory (the per-view targets;
    config 2 has none) and its result read device->host (the loss values; the rendered
    image for config 2), copies inside the timed region.  Returns (ms, views, h2d, d2h)."""
    import torch

    from paper_2501_18630_b200 import distributed as dd
    from paper_2501_18630_b200.rasterizer import check_pending, render_backward, render_tiled
    from paper_2501_18630_b200.training import AdamState, LossWorkspace, adam_step, group_lrs, loss_into

    prims, cams, bg = w["prims"], w["cams"], w["bg"]
    train = w["kind"] == "train"
    main = torch.cuda.current_stream()
    if train:
        if "e2e_host" not in w:  # pinned (torch.empty(pin_memory=True)) and exercised once
            w["e2e_host"] = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t.cpu())
                             for t in w["targets"]]
        host = w["e2e_host"]
        # two device copies of the targets: step i+1's upload (copy stream) overlaps step i
        tgt2 = [[torch.empty_like(t) for t in w["targets"]] for _ in range(2)]
        cs = torch.cuda.Stream()
        up_ev = [torch.cuda.Event(), torch.cuda.Event()]
        used_ev = [torch.cuda.Event(), torch.cuda.Event()]
        ws = {}
        for cam in cams:
            ws.setdefault((cam.width, cam.height), LossWorkspace(cam.width, cam.height))
        d_img = {k: torch.empty((k[1], k[0], 3), dtype=torch.float32, device="cuda") for k in ws}
        vals = torch.zeros((len(cams), 3), dtype=torch.float64, device="cuda")
        vals_host = torch.empty_like(vals, device="cpu").pin_memory()
        state = AdamState(prims) if w["adam"] else None
        lrs = group_lrs()
        bi = sum(h.numel() * h.element_size() for h in host)
        bo = vals.numel() * vals.element_size()
    else:
        side = torch.cuda.Stream()
        c0 = cams[0]
        img_host = [torch.empty((c0.height, c0.width, 3), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        bi, bo = 0, img_host[0].numel() * 4

    def step(i):
        if not train:
            out = render_tiled(prims, cams[0], bg)
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            out.color.record_stream(side)
            with torch.cuda.stream(side):  # frame i downloads while frame i+1 renders
                img_host[i % 2].copy_(out.color, non_blocking=True)
            return 1
        b = i % 2
        if i == 0:  # the first step's inputs (later ones were prefetched by the previous step)
            with torch.cuda.stream(cs):
                for v in range(len(cams)):
                    tgt2[0][v].copy_(host[v], non_blocking=True)
                up_ev[0].record(cs)
        with torch.cuda.stream(cs):  # prefetch step i+1's inputs once step i-1 released the buffer
            cs.wait_event(used_ev[b ^ 1])
            for v in range(len(cams)):
                tgt2[b ^ 1][v].copy_(host[v], non_blocking=True)
            up_ev[b ^ 1].record(cs)
        main.wait_event(up_ev[b])
        tgt = tgt2[b]
        grads = None  # the first view's backward writes a fresh buffer, later views add into it
        for v, cam in enumerate(cams):
            out = render_tiled(prims, cam, bg)
            k = (cam.width, cam.height)
            loss_into(out.color, tgt[v], d_img[k], ws[k], values=vals[v])
            grads = render_backward(prims, cam, bg, d_img[k], forward_out=out, grads=grads)
        if world > 1:
            dd.allreduce_grads(grads.flat)
        if state is not None:
            adam_step(prims, grads, state, lrs, device_step=True)
        used_ev[b].record(main)
        vals_host.copy_(vals, non_blocking=True)
        return len(cams)

    for i in range(3):  # untimed: allocator / capacity warm-up
        step(i)
    torch.cuda.synchronize()
    if train:  # the timed loop starts from step 0 again (no upload in flight)
        for ev in used_ev:
            ev.record(main)
    check_pending(block=True)
    warm_host_link()
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(main)
    views = 0
    for i in range(steps):
        views += step(i)
    main.wait_stream(side if not train else cs)  # the last prefetch / download is part of the run
    e.record(main)
    e.synchronize()
    ms = s.elapsed_time(e)
    check_pending(block=True)  # any device-side error / overflow invalidates the run
    barrier(world)
    return ms, views, bi, bo


def warm_host_link():
    """Bring host<->device copies to steady state before a timed region: on these boxes
    they start at ~11 GB/s and reach ~54 GB/s only after about a second of traffic."""
    import torch

    warm_dev = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
    warm_host = torch.empty(16 << 20, dtype=torch.uint8, pin_memory=True)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        for _ in range(8):
            warm_dev.copy_(warm_host, non_blocking=True)
            warm_host.copy_(warm_dev, non_blocking=True)
        torch.cuda.synchronize()


def deterministic_cost(w, reps=3):
    """Device time of one view's backward in the default mode vs the deterministic mode
    (bsr_backward_deterministic: fixed-point accumulation, two raster passes), on the
    step's own frame and upstream gradient (extra.deterministic_backward)."""
    import torch

    from paper_2501_18630_b200.rasterizer import backward_raw, det_workspace

    st = w.get("step")
    if st is None:
        return None
    cam = w["cams"][0]
    key = (cam.width, cam.height)
    frame, d_img = st.frames[key], st.bufs[key]["d_image"]
    ws = det_workspace(len(w["prims"]))
    out = {}
    for name, det in (("default_ms", None), ("deterministic_ms", ws)):
        backward_raw(st.scene, cam, w["bg"], frame, d_img, None, st.gc, det_ws=det)  # warm
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            backward_raw(st.scene, cam, w["bg"], frame, d_img, None, st.gc, det_ws=det)
        e.record()
        e.synchronize()
        out[name] = round(s.elapsed_time(e) / reps, 4)
    st.grads.flat.zero_()
    st._grads_clear = True
    del ws
    return out


# ----------------------------------------------------------------------------- peaks
def fp32_peaks(clk_mhz):
    """Measured FFMA / FFMA2 / SFU rates (profiles/r02_peaks.json, written by
    profiles/micro/run_peaks.py on this pool's B200), else the nominal FMA rate."""
    pk = peaks()
    nominal = SM_COUNT * FP32_LANES_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    try:
        with open(os.path.join(REPO, "profiles", "r02_peaks.json")) as f:
            m = json.load(f)
        return dict(fp32=max(float(m["ffma_tflops"]), float(m["ffma2_tflops"])), ffma2=float(m["ffma2_tflops"]),
                    sfu_gops=float(m["ex2_gops"]),
                    nominal=nominal, source=f"measured: profiles/micro/peaks.cu (best of FFMA / FFMA2 chains, 148x8 CTAs, "
                                            f"SM clock {m.get('sm_mhz_median')} MHz) -> profiles/r02_peaks.json")
    except Exception:
        return dict(fp32=nominal, ffma2=nominal, sfu_gops=None, nominal=nominal,
                    source="nominal FP32 FMA rate 148 SM x 128 lanes x 2 x sm_max_mhz")


# ----------------------------------------------------------------------------- one workload
def measure(cfg, args, rank, world, local, K, W, want_cpu, want_e2e):
    """Device-timed value, e2e, roofline and CPU baseline of one workload; returns the line."""
    import torch

    from paper_2501_18630_b200.rasterizer import frame_status

    w = build_b200(cfg, rank, world, args.views_per_gpu)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2
    for _ in range(W):  # warm-up (also sizes the tile-entry capacity with a checked forward)
        run_step(w)
    torch.cuda.synchronize()
    frames = [w["frame"]] if w["kind"] == "render" else list(w["step"].frames.values())
    for f in frames:
        frame_status(f)

    prof = BenchProfiler(len(w["cams"]))
    prof.sp.count_pairs(True)  # algorithmic pair counts (P_f, P_b) from one untimed step
    run_step(w, prof)
    torch.cuda.synchronize()
    pair_stats = prof.sp.stats.cpu().numpy().astype(np.float64) / len(w["cams"])
    prof.sp.count_pairs(False)
    prof.sp.collect_step()
    prof.sp.reset()
    # per-stage kernel durations: eager steps with libbsr's stage events (kernel time is the
    # same in and out of a graph; events cannot be timed inside a replayed graph)
    timed_loop(w, min(K, 20), world, prof=prof, l2=l2)
    timed_prof = prof
    if not args.eager:
        try:
            make_graph(w, None)
            timed_prof = None
        except Exception as exc:  # NCCL inside a capture is a driver/library feature: degrade, do not fail
            if world == 1:
                raise
            print(f"[bench] rank {rank}: graph capture with the all-reduce failed ({exc!r}); timing eager steps",
                  file=sys.stderr)
            w.pop("graph", None)
            torch.cuda.synchronize()
    if timed_prof is not None:
        prof.sp.reset()
    clocks = ClockSampler(local)
    clocks.start()
    ms, views = timed_loop(w, K, world, prof=timed_prof, l2=l2)
    clk = clocks.stop()
    for f in frames:  # any device-side error or capacity overflow invalidates the run
        frame_status(f)
    ms_max = max_over_ranks(ms, world)
    views_all = sum_over_ranks(views, world)
    value = views_all / (ms_max / 1e3)

    e2e = extra_e2e = None
    if want_e2e:
        ke = max(K, 10)
        try:
            ems, eviews, bi, bo = e2e_api_loop(w, ke, world)
            ems_max = max_over_ranks(ems, world)
            e2e = {"value": sum_over_ranks(eviews, world) / (ems_max / 1e3), "unit": unit_for(cfg),
                   "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(bo),
                   "path": "public API per step: render_tiled, training.loss_into, render_backward "
                           "(+ all-reduce + adam_step), eager; each step's inputs copied H2D from pinned "
                           "memory on a copy stream while the previous step computes (double-buffered), "
                           "the loss values read back D2H (config 2: render_tiled + the image D2H on a "
                           "side stream)"}
        except Exception as exc:
            if world == 1:
                raise
            print(f"[bench] rank {rank}: e2e failed ({exc!r})", file=sys.stderr)
        try:  # the same step captured with its copies in CUDA graphs (a serving / training loop's form)
            gms, gviews, gbi, gbo = e2e_loop(w, max(K, 20), world)
            gms_max = max_over_ranks(gms, world)
            extra_e2e = {"value": sum_over_ranks(gviews, world) / (gms_max / 1e3), "unit": unit_for(cfg),
                         "h2d_bytes_per_step": int(gbi), "d2h_bytes_per_step": int(gbo),
                         "path": "training.TrainStep / render step captured with its copies in two CUDA graphs"}
        except Exception as exc:
            print(f"[bench] rank {rank}: graph e2e failed ({exc!r})", file=sys.stderr)
            torch.cuda.synchronize()

    stages = prof.sp.mean_ms()
    pk = peaks()
    clk_mhz = clk.get("sm_mhz") or pk["sm_max_mhz"]
    fp = fp32_peaks(clk_mhz)
    pairs_f, contrib_f, pairs_b = pair_stats[0], pair_stats[1], pair_stats[2]
    rf = dict(raster_fwd=(pairs_f * FP32_FLOP_PER_PAIR_FWD, stages["raster_fwd"]))
    if w["kind"] == "train":
        rf["raster_bwd"] = (pairs_b * FP32_FLOP_PER_PAIR_BWD, stages["raster_bwd"])
    per_view = {k: v for k, v in stages.items() if k not in ("adam", "color_views")}
    dom = max(per_view, key=lambda k: per_view[k])
    extra = {"stage_ms": {k: round(v, 4) for k, v in stages.items()},
             "pairs_per_view": {"fwd": pairs_f, "bwd": pairs_b, "contributions": contrib_f},
             "dominant_stage": dom}
    ach = {}
    for k, (flop, t_ms) in rf.items():
        a = flop / (t_ms * 1e-3) / 1e12
        ach[k] = {"achieved_tflops": round(a, 3), "frac_of_measured_ffma": round(a / fp["fp32"], 4),
                  "frac_of_nominal": round(a / fp["nominal"], 4)}
    extra["raster_roofline"] = ach
    nscene = len(w["prims"])
    k3 = w["prims"].sh_coeffs
    info = frames[0].info
    V, E = info["visible"], info["entries"]
    hbm = {}
    hbm["preprocess"] = (nscene * (48 + 12 * k3) + V * 80 + E * 4) / (stages["preprocess"] * 1e-3) / 1e9
    n_tiles = (-(-w["cams"][0].width // 16)) * (-(-w["cams"][0].height // 16))
    hbm["bin_count"] = (n_tiles * 12) / (stages["bin_count"] * 1e-3) / 1e9
    hbm["bin_scatter"] = (V * 24 + E * 12) / (stages["bin_scatter"] * 1e-3) / 1e9
    hbm["tile_sort"] = (E * 12) / (stages["tile_sort"] * 1e-3) / 1e9
    if w["kind"] == "train":
        # geometry chain (fp64 kernel) + colour chain: grad_acc 48 + params 240 + gradients
        # RMW 480 per visible primitive at SH-3; with the colour chain deferred to color_views
        # grad_acc 48 + geometry params 48 + their gradients RMW 96 + d rgb 16
        per_vis = 208 if stages.get("color_views", 0) > 0 else (48 + 240 + 480)
        hbm["preprocess_bwd"] = V * per_vis / (stages["preprocess_bwd"] * 1e-3) / 1e9
        cam0 = w["cams"][0]
        if stages.get("loss", 0) > 0:
            hbm["loss"] = 12 * 3 * cam0.width * cam0.height * 4 / (stages["loss"] * 1e-3) / 1e9
        if stages.get("color_views", 0) > 0:
            nv = len(w["cams"])
            hbm["color_views"] = nscene * (12 * k3 * 3 + 16 * nv + 12) / (stages["color_views"] * 1e-3) / 1e9
        if stages.get("adam", 0) > 0:
            hbm["adam"] = 28 * w["prims"].flat.numel() / (stages["adam"] * 1e-3) / 1e9
    extra["hbm_stage_gbs"] = {k: round(v, 1) for k, v in hbm.items()}
    extra["visible"], extra["entries"], extra["flagged_pixels"] = V, E, info["flagged_pixels"]
    if dom in rf:
        flop, t_ms = rf[dom]
        a = flop / (t_ms * 1e-3) / 1e12
        roof = {"bound": "fp32", "achieved": round(a, 3), "peak": round(fp["fp32"], 2), "unit": "TFLOP/s",
                "frac": round(a / fp["fp32"], 4), "traffic": None, "kernel": dom, "peak_source": fp["source"],
                "nominal_peak": round(fp["nominal"], 2), "ffma2_peak": round(fp["ffma2"], 2),
                "algorithmic": f"{FP32_FLOP_PER_PAIR_FWD if dom == 'raster_fwd' else FP32_FLOP_PER_PAIR_BWD} "
                               f"FLOP per evaluated (pixel, entry) pair (SURVEY 8(d)) x pairs counted on the "
                               f"device in an untimed step / the kernel's mean CUDA-event duration"}
    else:
        gbs = hbm.get(dom)
        roof = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": None if gbs is None else gbs / pk["hbm_gbs"], "traffic": None, "kernel": dom}
    ncu = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(ncu):
        try:
            tr = json.load(open(ncu)).get(cfg, {}).get(roof["kernel"])
            if tr:
                roof["traffic"] = tr
        except Exception:
            pass
    cam = w["cams"][0]
    line = {
        "metric": metric_for(cfg), "value": value, "unit": unit_for(cfg), "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "strong" if cfg == "c3" else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded BASELINE config generators, random-init Gaussians)",
        "config": {"workload": cfg, "gaussians": len(w["prims"]), "sh_degree": 3, "width": cam.width,
                   "height": cam.height, "views_per_gpu": len(w["cams"]),
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": "flushed between steps (256 MiB write)"},
        "roofline": roof, "cpu_baseline": None, "e2e": e2e,
        "gpu_launches": kernel_launches_per_step(w) * K, "clocks": clk, "extra": extra,
        "cuda_graph": "graph" in w,
    }
    if extra_e2e is not None:
        line["extra"]["e2e_graph"] = extra_e2e
    if w["kind"] == "train" and world == 1:
        try:
            line["extra"]["deterministic_backward"] = deterministic_cost(w)
        except Exception as exc:
            print(f"[bench] deterministic timing failed ({exc!r})", file=sys.stderr)
    if world > 1:
        line["nccl"] = nccl_info()
    del w, l2
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if want_cpu and rank == 0 and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as e:  # the baseline is reported, never the target
            line["cpu_baseline"] = {"value": None, "unit": unit_for(cfg), "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"unavailable: {e!r}"}
    return line


def nccl_info():
    import torch
    import torch.distributed as dist

    try:
        ver = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        ver = None
    return {"backend": dist.get_backend(), "world_size": dist.get_world_size(), "nccl_version": ver,
            "collective": "per step: reduce_scatter (sum, fp32) of the flat per-Gaussian gradient buffer, "
                          "Adam on the rank's shard, all_gather of the parameter shards "
                          "(distributed.ShardedOptimizer); e2e: all_reduce + adam_step through the API"}


# ----------------------------------------------------------------------------- launcher
def spawn_ranks(n):
    """`bench.py --gpus N` without a torchrun environment: relaunch this command under
    torch.distributed.run with N local ranks (one per GPU, NCCL, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (rank count) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4"],
                    help="default: c4 (the largest single-GPU config) at N=1, c3 (view-batch DP) at N>1")
    ap.add_argument("--views-per-gpu", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-1 line nested in the c4 line")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph capture of the step")
    args = ap.parse_args()
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)  # does not return
    if args.config is None:
        args.config = "c4" if max(world_env, 1) == 1 else "c3"
    if args.impl == "reference":
        return run_reference(args)

    import torch

    rank, world, local = dist_setup(args.gpus)
    from paper_2501_18630_b200 import _lib

    _lib.require_cuda()
    W = max(args.warmup, 3)
    K = max(args.steps, 1)
    line = measure(args.config, args, rank, world, local, K, W, not args.no_cpu_baseline, not args.no_e2e)
    if world == 1 and args.config == "c4" and not args.no_secondary:
        # config 1 (the reference's CPU-sized training step) as a secondary figure
        sec = measure("c1", args, rank, world, local, max(K, 20), W, not args.no_cpu_baseline, not args.no_e2e)
        line["secondary"] = {"c1": {k: sec[k] for k in ("metric", "value", "unit", "ms_per_step", "e2e", "roofline",
                                                          "cpu_baseline", "clocks")}}
        line["secondary"]["c1"]["stage_ms"] = sec["extra"]["stage_ms"]
        line["secondary"]["c1"]["e2e_graph"] = sec["extra"].get("e2e_graph")
        line["gpu_launches_secondary"] = sec["gpu_launches"]
        # config 3 at one GPU: the base of the multi-GPU series (the N > 1 default is config 3,
        # N = 1 is config 4), so scaling efficiency can be read off the same config
        base = measure("c3", args, rank, world, local, 5, W, False, False)
        line["scaling_base"] = {"workload": "c3", "value": base["value"], "unit": base["unit"],
                                "ms_per_step": base["ms_per_step"], "n_gpus": 1,
                                "note": "config 3 (32 views, 3M Gaussians) on this one GPU; bench.py --gpus N (N > 1) "
                                        "measures config 3 split 32/N across N GPUs"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
