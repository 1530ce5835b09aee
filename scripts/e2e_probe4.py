"""Mimic bench.main() for config 1 up to the e2e loop, then time e2e variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2501_18630_b200.rasterizer import frame_status

early_host = torch.empty(800 * 800 * 3, dtype=torch.float32, pin_memory=True)
w = bench.build_b200("c1", 0, 1, 1)
early_host.copy_(w["targets"][0].reshape(-1).cpu())
l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    bench.run_step(w)
torch.cuda.synchronize()
for f in w["step"].frames.values():
    frame_status(f)
prof = bench.BenchProfiler(1)
prof.sp.count_pairs(True); bench.run_step(w, prof); torch.cuda.synchronize(); prof.sp.count_pairs(False)
prof.sp.collect_step(); prof.sp.reset()
bench.timed_loop(w, 20, 1, prof=prof, l2=l2)
bench.make_graph(w, None)
ms, v = bench.timed_loop(w, 50, 1, prof=None, l2=l2)
print(f"device loop: {ms/50*1e3:.1f} us/step")
for r in range(3):
    ms, views, bi, bo = bench.e2e_loop(w, 50, 1)
    print(f"e2e_loop #{r}: {ms/50*1e3:.1f} us/step")
del l2
torch.cuda.empty_cache()
ms, views, bi, bo = bench.e2e_loop(w, 50, 1)
print(f"e2e_loop after freeing the L2 flush buffer: {ms/50*1e3:.1f} us/step")

# inline pipeline (as e2e_probe3) in this state
K = 50
host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t.cpu()) for t in w["targets"]]
stage = [[torch.empty_like(t) for t in w["targets"]] for _ in range(2)]
res_dev = w["step"].loss_values
res_host = [torch.empty(res_dev.shape, dtype=res_dev.dtype, pin_memory=True) for _ in range(2)]
cs = torch.cuda.Stream()
g0 = w.pop("graph")
gs = []
for b in range(2):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            for dst, h in zip(stage[b ^ 1], host):
                dst.copy_(h, non_blocking=True)
        for dst, src in zip(w["targets"], stage[b]):
            dst.copy_(src, non_blocking=True)
        bench.run_step(w)
        res_host[b].copy_(res_dev, non_blocking=True)
        cur.wait_stream(cs)
    gs.append(g)
def run(gs, label):
    done = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(K):
        gs[i % len(gs)].replay()
        done[i % 2].record()
        if i >= 1:
            done[(i - 1) % 2].synchronize()
    e.record(); e.synchronize()
    print(f"{label}: {s.elapsed_time(e)/K*1e3:.1f} us/step")
run(gs, "inline pipeline")
run(gs, "inline pipeline again")
w["graph"] = g0
def seq():
    for i in range(K):
        w["graph"].replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); seq(); e.record(); e.synchronize()
print(f"plain graph replay: {s.elapsed_time(e)/K*1e3:.1f} us/step")
g0 = w.pop("graph")
def cap(h2d, d2d, d2h):
    gs = []
    for b in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cur = torch.cuda.current_stream()
            if h2d:
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
            if h2d:
                cur.wait_stream(cs)
        gs.append(g)
    return gs
for args in ((False, False, False), (True, False, False), (False, True, False), (False, False, True)):
    run(cap(*args), f"recaptured step h2d/d2d/d2h={args}")

host_saved = host
host = [early_host.view(800, 800, 3)]
run(cap(True, False, False), "recaptured step + H2D from a pinned buffer allocated at start")
host = [torch.empty((800, 800, 3), dtype=torch.float32, pin_memory=True)]
run(cap(True, False, False), "recaptured step + H2D from a freshly pinned buffer")
import ctypes
host = host_saved
run(cap(True, False, False), "recaptured step + H2D from the first e2e host buffer, again at the end")
for r in range(2):
    ms, views, bi, bo = bench.e2e_loop(w, 50, 1)
    print(f"e2e_loop at the end #{r}: {ms/50*1e3:.1f} us/step")
