# Diagnostic (needs a library built with EXTRA=-DBSR_FLAG_REASONS): why the fp32 raster
# hands pixels to the fp64 replay, per config.  python scripts/gpu/flag_reasons.py c4 c3 c1
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_18630_b200 import _lib  # noqa: E402

lib = _lib.load()
fn = lib.bsr_debug_flag_reasons
for cfg in sys.argv[1:]:
    w = bench.build_b200(cfg, 0, 1, 32 if cfg == "c3" else 1)
    bench.run_step(w)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 6)()
    fn(out, 1)
    bench.run_step(w)
    torch.cuda.synchronize()
    fn(out, 1)
    print(cfg, "alpha_cut", out[0], "alpha>0.999", out[1], "T_stop", out[2], "| fp32", out[3], "needle", out[4],
          "fp64", out[5], flush=True)
    del w
    torch.cuda.empty_cache()
