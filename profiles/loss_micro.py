import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2501_18630_b200.training import LossWorkspace, loss_into
for (w, h) in [(800, 800), (1600, 1067)]:
    a = torch.rand(h, w, 3, device='cuda'); b = torch.rand(h, w, 3, device='cuda'); d = torch.empty_like(a)
    ws = LossWorkspace(w, h)
    for _ in range(5): loss_into(a, b, d, ws)
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(100): loss_into(a, b, d, ws)
    e.record(); e.synchronize()
    print(w, h, 'loss ms', s.elapsed_time(e) / 100)
