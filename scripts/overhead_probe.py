"""Graph-replayed training step at tiny sizes: the floor set by kernel boundaries."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_18630_b200 import PrimitiveSet
from paper_2501_18630_b200.scenes import make_workload, target_scene
from paper_2501_18630_b200.training import TrainStep, render_targets

SIZES = ((1000, 64, 64), (10000, 256, 256), (100000, 800, 800))
if len(sys.argv) > 1:  # e.g. `tiny` -> the first size only, few replays (for ncu)
    SIZES = SIZES[:1]
for n, w, h in SIZES:
    wl = make_workload("c1", seed=0, n=n, width=w, height=h)
    prims = PrimitiveSet.from_scene(wl.scene)
    tgt = PrimitiveSet.from_scene(target_scene("c1", 1, n))
    targets = render_targets(tgt, wl.cameras, wl.background)
    st = TrainStep(prims, wl.cameras, targets, wl.background)
    st.step(check=True)
    g = st.capture()
    for _ in range(10):
        st.replay()
    torch.cuda.synchronize()
    K = 200 if len(sys.argv) == 1 else 3
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(K):
        st.replay()
    e.record(); e.synchronize()
    print(f"n={n} {w}x{h}: {s.elapsed_time(e)/K*1e3:.1f} us/step")
