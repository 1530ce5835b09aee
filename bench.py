"""Benchmark of the hot path (BASELINE.json metric: render FPS / train it/s on B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4]
    python bench.py --impl reference ...      (the reference's CPU implementation)

Default workload (N=1): BASELINE config 1 -- one training step = forward render of
N=100k SH-3 Gaussians at 800x800 + 0.8 L1 + 0.2 D-SSIM loss + backward + Adam, all on the
device through libbsr.so.  With N>1 (torchrun, NCCL) every rank trains on its own view of
the same scene (weak scaling: one 800x800 view per GPU per step) and the flat per-Gaussian
gradient buffer is all-reduced before Adam.  --config c3 runs the 32-view batch of
config 3 split across ranks (strong scaling), c2 the 1080p forward render, c4 the 4K
stress forward + backward.

Timing: W warm-up steps, then K steps each timed with CUDA events on the launching
stream (L2 flushed with a 256 MiB write between steps, outside the events), bracketed by
barrier + synchronize, max over ranks.  Stage times / pair counts for the roofline come
from libbsr's caller-owned events and device counters recorded inside the same timed
steps.  e2e repeats the step through the public API with the per-step inputs (target
images) copied from pinned host memory and the loss read back, copies inside the timing.
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
    from paper_2501_18630_b200 import distributed as dd

    return dd.init("nccl" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else None)


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
    """Same step through the public API with per-step host inputs (pinned) and the result
    read back, copies inside the timing.

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
    # steady-state host link: on the B200 boxes host<->device copies start at ~11 GB/s and
    # reach ~54 GB/s only after about a second of sustained traffic (scripts/h2d_probe.py,
    # scripts/e2e_probe4.py); bring the link up before timing, as a running job would have
    warm_dev = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
    warm_host = torch.empty(16 << 20, dtype=torch.uint8, pin_memory=True)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        for _ in range(8):
            warm_dev.copy_(warm_host, non_blocking=True)
            warm_host.copy_(warm_dev, non_blocking=True)
        torch.cuda.synchronize()
    del warm_dev, warm_host

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
    step()  # warm-up (first-touch, BLAS init)
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
    warm = min(args.warmup, 1)
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


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c1", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--views-per-gpu", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph capture of the step")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    rank, world, local = dist_setup(args.gpus)
    from paper_2501_18630_b200 import _lib

    _lib.require_cuda()
    W = max(args.warmup, 3)
    K = max(args.steps, 1)
    w = build_b200(args.config, rank, world, args.views_per_gpu)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    # warm-up (also sizes the tile-entry capacity with a checked forward)
    from paper_2501_18630_b200.rasterizer import frame_status

    for _ in range(W):
        run_step(w)
    torch.cuda.synchronize()
    frames = [w["frame"]] if w["kind"] == "render" else list(w["step"].frames.values())
    for f in frames:
        frame_status(f)

    prof = BenchProfiler(len(w["cams"]))
    if prof is not None:  # algorithmic pair counts (P_f, P_b) from one untimed step
        prof.sp.count_pairs(True)
        run_step(w, prof)
        torch.cuda.synchronize()
        pair_stats = prof.sp.stats.cpu().numpy().astype(np.float64) / len(w["cams"])
        prof.sp.count_pairs(False)
        prof.sp.collect_step()
        prof.sp.reset()
    timed_prof = prof
    if not args.eager:
        # per-stage kernel durations: eager steps with libbsr's stage events (kernel time is
        # the same in and out of a graph; events cannot be timed inside a replayed graph)
        timed_loop(w, min(K, 20), world, prof=prof, l2=l2)
        try:
            make_graph(w, None)
        except Exception as exc:  # NCCL inside a capture is a driver/library feature: degrade, do not fail
            if world == 1:
                raise
            import sys as _sys

            print(f"[bench] rank {rank}: graph capture with the all-reduce failed ({exc!r}); "
                  f"timing eager steps", file=_sys.stderr)
            w.pop("graph", None)
            torch.cuda.synchronize()
        timed_prof = None
    clocks = ClockSampler(local)
    clocks.start()
    ms, views = timed_loop(w, K, world, prof=timed_prof, l2=l2)
    clk = clocks.stop()
    for f in frames:  # any device-side error or capacity overflow invalidates the run
        frame_status(f)
    ms_max = max_over_ranks(ms, world)
    views_all = sum_over_ranks(views, world)
    value = views_all / (ms_max / 1e3)

    e2e = None
    if not args.no_e2e:
        ke = max(K, 20)
        try:
            ems, eviews, bi, bo = e2e_loop(w, ke, world)
        except Exception as exc:  # see the capture fallback above
            if world == 1:
                raise
            import sys as _sys

            print(f"[bench] rank {rank}: e2e capture failed ({exc!r})", file=_sys.stderr)
            torch.cuda.synchronize()
            ems = None
        if ems is not None:
            ems_max = max_over_ranks(ems, world)
            e2e = {"value": sum_over_ranks(eviews, world) / (ems_max / 1e3), "unit": unit_for(args.config),
                   "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(bo)}

    pk = peaks()
    roof, stages, extra = None, None, {}
    if prof is not None:
        stages = prof.sp.mean_ms()
        pairs_f, contrib_f, pairs_b = pair_stats[0], pair_stats[1], pair_stats[2]
        clk_mhz = clk.get("sm_mhz") or pk["sm_max_mhz"]
        fp32_peak_max = SM_COUNT * FP32_LANES_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        fp32_peak_clk = SM_COUNT * FP32_LANES_PER_SM * 2 * clk_mhz * 1e6 / 1e12
        rf = dict(raster_fwd=(pairs_f * FP32_FLOP_PER_PAIR_FWD, stages["raster_fwd"]))
        if w["kind"] == "train":
            rf["raster_bwd"] = (pairs_b * FP32_FLOP_PER_PAIR_BWD, stages["raster_bwd"])
        # dominant per-view stage (adam / color_views run once per multi-view step)
        per_view = {k: v for k, v in stages.items() if k not in ("adam", "color_views")}
        dom = max(per_view, key=lambda k: per_view[k])
        extra["stage_ms"] = {k: round(v, 4) for k, v in stages.items()}
        extra["pairs_per_view"] = {"fwd": pairs_f, "bwd": pairs_b, "contributions": contrib_f}
        extra["dominant_stage"] = dom
        ach = {}
        for k, (flop, t_ms) in rf.items():
            a = flop / (t_ms * 1e-3) / 1e12
            ach[k] = {"achieved_tflops": round(a, 3), "frac_of_fp32_peak_at_max_clock": round(a / fp32_peak_max, 4),
                      "frac_of_fp32_peak_at_measured_clock": round(a / fp32_peak_clk, 4)}
        extra["raster_roofline"] = ach
        # HBM stages: algorithmic bytes / stage time
        nscene = len(w["prims"])
        k3 = w["prims"].sh_coeffs
        info = frames[0].info
        V, E = info["visible"], info["entries"]
        hbm = {}
        # preprocess: parameters (geometry 48 B + SH 12 K B), records 80 B per visible, and the
        # per-tile counts (E 4-B REDs, taken here since the counting pass was fused in)
        hbm["preprocess"] = (nscene * (48 + 12 * k3) + V * 80 + E * 4) / (stages["preprocess"] * 1e-3) / 1e9
        # binning: scan = T counts read + T ranges written (12 B); scatter = V (20 B + key
        # 4 B) + E (8-B entry + 4-B atomic); per-tile sort = E (8 B read + 4 B written)
        n_tiles = frames[0].info.get("tiles") or (-(-w["cams"][0].width // 16)) * (-(-w["cams"][0].height // 16))
        hbm["bin_count"] = (n_tiles * 12) / (stages["bin_count"] * 1e-3) / 1e9
        hbm["bin_scatter"] = (V * 24 + E * 12) / (stages["bin_scatter"] * 1e-3) / 1e9
        hbm["tile_sort"] = (E * 12) / (stages["tile_sort"] * 1e-3) / 1e9
        if w["kind"] == "train":
            # geometry chain + colour chain (768 B / visible primitive at SH-3); with the colour
            # chain deferred to color_views: grad_acc 48 + geometry params 48 + their
            # gradients read-modify-write 96 + d rgb 16
            per_vis = 208 if stages.get("color_views", 0) > 0 else (48 + 240 + 480)
            hbm["preprocess_bwd"] = V * per_vis / (stages["preprocess_bwd"] * 1e-3) / 1e9
            cam0 = w["cams"][0]
            if stages.get("loss", 0) > 0:
                hbm["loss"] = 12 * 3 * cam0.width * cam0.height * 4 / (stages["loss"] * 1e-3) / 1e9
            if stages.get("color_views", 0) > 0:  # once per step: SH rows read, gradients RMW
                nv = len(w["cams"])
                hbm["color_views"] = nscene * (12 * k3 * 3 + 16 * nv + 12) / (stages["color_views"] * 1e-3) / 1e9
            if stages.get("adam", 0) > 0:
                hbm["adam"] = 28 * w["prims"].flat.numel() / (stages["adam"] * 1e-3) / 1e9
        extra["hbm_stage_gbs"] = {k: round(v, 1) for k, v in hbm.items()}
        extra["visible"], extra["entries"], extra["flagged_pixels"] = V, E, info["flagged_pixels"]
        if dom in rf:
            flop, t_ms = rf[dom]
            a = flop / (t_ms * 1e-3) / 1e12
            roof = {"bound": "fp32", "achieved": round(a, 3), "peak": round(fp32_peak_max, 2), "unit": "TFLOP/s",
                    "frac": round(a / fp32_peak_max, 4), "traffic": None, "kernel": dom,
                    "peak_source": "nominal FP32 FMA rate 148 SM x 128 lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json "
                                   "has no FP32 figure; the raster is not a dense contraction, no tensor cores)",
                    "algorithmic": f"{FP32_FLOP_PER_PAIR_FWD if dom == 'raster_fwd' else FP32_FLOP_PER_PAIR_BWD} "
                                   f"FLOP per evaluated (pixel, entry) pair x pairs counted on device"}
        else:
            gbs = hbm.get(dom)
            roof = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": None if gbs is None else gbs / pk["hbm_gbs"], "traffic": None, "kernel": dom}
        ncu = os.path.join(REPO, "profiles", "ncu_traffic.json")
        if os.path.exists(ncu) and roof is not None:
            try:
                tr = json.load(open(ncu)).get(args.config, {}).get(roof["kernel"])
                if tr:
                    roof["traffic"] = tr
            except Exception:
                pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config)
        except Exception as e:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": unit_for(args.config), "cores": os.cpu_count(), "kind": "port",
                   "sample": f"unavailable: {e!r}"}

    if rank == 0:
        cam = w["cams"][0]
        line = {
            "metric": metric_for(args.config), "value": value, "unit": unit_for(args.config), "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
            "scaling": "strong" if args.config == "c3" else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE config generators, random-init Gaussians)",
            "config": {"workload": args.config, "gaussians": len(w["prims"]), "sh_degree": 3,
                       "width": cam.width, "height": cam.height, "views_per_gpu": len(w["cams"]),
                       "parallelism": f"dp{world}" if world > 1 else "single", "l2": "flushed between steps"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": kernel_launches_per_step(w) * K, "clocks": clk, "extra": extra,
            "cuda_graph": "graph" in w,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
