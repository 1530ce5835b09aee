# Host-side profile of the public-API step (bench.py e2e_api_loop) at a config: where the
# Python time per step goes.  python scripts/gpu/prof_e2e.py c1
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = bench.build_b200(cfg, 0, 1, 32 if cfg == "c3" else 1)
bench.e2e_api_loop(w, 20, 1)
pr = cProfile.Profile()
pr.enable()
ms, views, _, _ = bench.e2e_api_loop(w, 200, 1)
pr.disable()
print(cfg, "ms per step", ms / 200)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumtime").print_stats(30)
