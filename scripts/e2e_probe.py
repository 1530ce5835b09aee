"""Probe where the config-1 e2e time goes (host-side overhead vs copies)."""
import sys, time, os
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
bench.make_graph(w)
K = 200
def timeit(fn, label):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    fn()
    e.record(); e.synchronize()
    t1 = time.perf_counter()
    print(f"{label}: device {s.elapsed_time(e)/K*1e3:.1f} us/step, host {1e6*(t1-t0)/K:.1f} us/step")
def graph_only():
    for _ in range(K):
        w["graph"].replay()
timeit(graph_only, "graph replay only")
def graph_sync():
    for _ in range(K):
        w["graph"].replay()
        torch.cuda.current_stream().synchronize()
timeit(graph_sync, "graph + sync each step")
def e2e():
    bench.e2e_loop(w, K, 1)
timeit(e2e, "bench.e2e_loop")
host = [t.cpu().pin_memory() for t in w["targets"]]
def h2d_only():
    for _ in range(K):
        for d, h in zip(w["targets"], host):
            d.copy_(h, non_blocking=True)
timeit(h2d_only, "H2D 7.7 MB only")
