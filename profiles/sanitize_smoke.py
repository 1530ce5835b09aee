"""Small end-to-end run exercising every libbsr kernel (for compute-sanitizer)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_18630_b200 import PrimitiveSet, backend, render_backward, render_tiled  # noqa: E402
from paper_2501_18630_b200.camera import Camera  # noqa: E402
from paper_2501_18630_b200.scenes import make_workload, sb_random_scene, target_scene  # noqa: E402
from paper_2501_18630_b200.training import TrainStep, render_targets  # noqa: E402

wl = make_workload("c4", seed=0, n=20_000, width=333, height=197)  # near-plane giants + big rects
prims = PrimitiveSet.from_scene(wl.scene)
out = render_tiled(prims, wl.cameras[0], wl.background)
g = render_backward(prims, wl.cameras[0], wl.background, np.random.default_rng(0).standard_normal(
    (197, 333, 3)).astype(np.float32), forward_out=out, d_depth=np.ones((197, 333), np.float32))
print("c4-like", out.frame.info)
sb = PrimitiveSet.from_reference(sb_random_scene(np.random.default_rng(1), 300, lobes=3))
cam = Camera.from_lookat((0.2, -0.3, -4.0), (0, 0, 0), (0, 1, 0), 0.9, 70, 50)
o2 = render_tiled(sb, cam, np.ones(3))
render_backward(sb, cam, np.ones(3), np.ones((50, 70, 3), np.float32), forward_out=o2)
wl1 = make_workload("c1", seed=0, n=5000, width=96, height=80)
tg = render_targets(PrimitiveSet.from_scene(target_scene("c1", 1, 5000)), wl1.cameras, wl1.background)
st = TrainStep(PrimitiveSet.from_scene(wl1.scene), wl1.cameras, tg, wl1.background)
st.step(check=True)
st.step()
# multi-view step (deferred colour chain), needles, codec round trip
cams = [Camera.from_lookat((np.sin(a) * 4.0, 0.3, -np.cos(a) * 4.0), (0, 0, 0), (0, 1, 0), 0.9, 72, 56)
        for a in np.linspace(-0.6, 0.6, 10)]
tg3 = render_targets(PrimitiveSet.from_scene(target_scene("c1", 1, 3000)), cams, wl1.background)
st3 = TrainStep(PrimitiveSet.from_scene(make_workload("c1", seed=0, n=3000).scene), cams, tg3, wl1.background)
st3.step(check=True)
nd = make_workload("c1", seed=3, n=600).scene
nd.log_scales[:300] = np.log(np.array([0.8, 0.004, 0.004], np.float32))
pn = PrimitiveSet.from_scene(nd)
on = render_tiled(pn, wl1.cameras[0], wl1.background)
render_backward(pn, wl1.cameras[0], wl1.background, np.ones((80, 96, 3), np.float32), forward_out=on)
import tempfile

from paper_2501_18630_b200 import compression

with tempfile.TemporaryDirectory() as d:
    compression.pack(sb, d)
    compression.unpack(d)
    compression.pack(pn, d + "/sh")
    compression.unpack(d + "/sh")
core = backend.get_core("cuda")
torch.cuda.synchronize()
print("sanitize smoke ok")
