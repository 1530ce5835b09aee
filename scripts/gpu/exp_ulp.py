# How often does CUDA's fp64 exp (torch float64 on the device) differ from numpy's exp (the
# reference's) on the scene parameters that feed the projection (log scales) and opacity?
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_18630_b200.scenes import make_workload  # noqa: E402

wl = make_workload("c4", seed=0)
for name, x in [("log_scales", np.asarray(wl.scene.log_scales, np.float64).ravel()),
                ("-opacity_raw", -np.asarray(wl.scene.opacity_raw, np.float64).ravel())]:
    a = np.exp(x)
    b = torch.exp(torch.from_numpy(x).cuda()).cpu().numpy()
    d = a != b
    ulps = np.abs(a.view(np.int64) - b.view(np.int64))
    print(f"{name}: n={x.size} numpy!=cuda {d.sum()} ({d.mean():.4%}), max ulps {ulps.max()}", flush=True)
