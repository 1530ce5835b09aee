"""Probe: H2D of the config-1 targets inside / beside the step graph."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

w = bench.build_b200("c1", 0, 1, 1)
for _ in range(5):
    bench.run_step(w)
torch.cuda.synchronize()
from paper_2501_18630_b200.rasterizer import frame_status
for f in w["step"].frames.values():
    frame_status(f)
K = 100
host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t.cpu()) for t in w["targets"]]
stage = [torch.empty_like(t) for t in w["targets"]]
cs = torch.cuda.Stream()
def timed(label, fn):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); e.synchronize()
    print(f"{label}: {s.elapsed_time(e)/K*1e3:.1f} us/step")
def mk(with_h2d, with_step, same_stream=False):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        if with_h2d:
            if same_stream:
                for d, h in zip(stage, host): d.copy_(h, non_blocking=True)
            else:
                cs.wait_stream(cur)
                with torch.cuda.stream(cs):
                    for d, h in zip(stage, host): d.copy_(h, non_blocking=True)
        if with_step:
            bench.run_step(w)
        if with_h2d and not same_stream:
            cur.wait_stream(cs)
    return g
for label, args in (("step only", (False, True)), ("h2d only (graph)", (True, False)),
                    ("h2d branch + step", (True, True)), ("h2d serial + step", (True, True, True))):
    g = mk(*args)
    timed(label, lambda g=g: [g.replay() for _ in range(K)])
def eager_h2d():
    for _ in range(K):
        for d, h in zip(stage, host): d.copy_(h, non_blocking=True)
timed("h2d only (eager)", eager_h2d)
print("host tensors pinned:", [h.is_pinned() for h in host], [h.numel() * 4 for h in host])
ms, views, bi, bo = bench.e2e_loop(w, K, 1)
print(f"bench.e2e_loop: {ms/K*1e3:.1f} us/step")
# e2e_loop without the per-step host sync
import types
src = open(os.path.join(os.path.dirname(bench.__file__), "bench.py")).read()
ms, views, bi, bo = bench.e2e_loop(w, K, 1)
print(f"bench.e2e_loop again: {ms/K*1e3:.1f} us/step")
