"""Probe variants of the e2e pipeline (config 1)."""
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
stage = [[torch.empty_like(t) for t in w["targets"]] for _ in range(2)]
res_dev = w["step"].loss_values
res_host = [torch.empty(res_dev.shape, dtype=res_dev.dtype, pin_memory=True) for _ in range(2)]
cs = torch.cuda.Stream()
def build(d2d=True, d2h=True, two=True):
    gs = []
    for b in range(2 if two else 1):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cur = torch.cuda.current_stream()
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                for dst, h in zip(stage[b ^ 1], host):
                    dst.copy_(h, non_blocking=True)
            if d2d:
                for dst, src in zip(w["targets"], stage[b]):
                    dst.copy_(src, non_blocking=True)
            bench.run_step(w)
            if d2h:
                res_host[b].copy_(res_dev, non_blocking=True)
            cur.wait_stream(cs)
        gs.append(g)
    return gs
def run(gs, sync=True, label=""):
    done = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(K):
        gs[i % len(gs)].replay()
        done[i % 2].record()
        if sync and i >= 1:
            done[(i - 1) % 2].synchronize()
    e.record(); e.synchronize()
    print(f"{label}: {s.elapsed_time(e)/K*1e3:.1f} us/step")
for kw, sync, label in (({}, True, "full"), ({}, False, "full, no host sync"), ({"d2h": False}, True, "no D2H"),
                        ({"d2d": False}, True, "no D2D"), ({"two": False}, True, "one graph"),
                        ({"d2h": False, "d2d": False}, True, "H2D branch only + sync")):
    gs = build(**kw)
    run(gs, sync, label)
    run(gs, sync, label + " (again)")
