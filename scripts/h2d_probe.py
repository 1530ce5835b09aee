"""Host->device bandwidth on this box for the e2e target upload (7.68 MB fp32 image)."""
import time
import torch

n = 800 * 800 * 3
dev = torch.empty(n, dtype=torch.float32, device="cuda")
K = 100
def bw(label, fn, nbytes):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); e.synchronize()
    ms = s.elapsed_time(e) / K
    print(f"{label}: {ms*1e3:.0f} us per copy, {nbytes/ms/1e6:.1f} GB/s")
for label, host in (("pin_memory()", torch.randn(n).pin_memory()),
                    ("empty(pin_memory=True)", torch.empty(n, pin_memory=True).normal_())):
    bw("H2D " + label, lambda h=host: [dev.copy_(h, non_blocking=True) for _ in range(K)], n * 4)
host = torch.empty(n, pin_memory=True).normal_()
streams = [torch.cuda.Stream() for _ in range(4)]
def split4():
    for _ in range(K):
        ev = torch.cuda.Event()
        ev.record()
        chunks = zip(dev.chunk(4), host.chunk(4))
        for st, (d, h) in zip(streams, chunks):
            st.wait_event(ev)
            with torch.cuda.stream(st):
                d.copy_(h, non_blocking=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
bw("H2D split over 4 streams", split4, n * 4)
hd = torch.empty(n, pin_memory=True)
bw("D2H", lambda: [hd.copy_(dev, non_blocking=True) for _ in range(K)], n * 4)
big = torch.empty(64 * n, pin_memory=True).normal_(); dbig = torch.empty(64 * n, device="cuda")
K2 = K; K = 5
bw("H2D 491 MB", lambda: [dbig.copy_(big, non_blocking=True) for _ in range(5)], 64 * n * 4)
