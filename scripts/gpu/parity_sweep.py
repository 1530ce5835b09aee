# Extra full-size parity cases beyond the pytest suite (other seeds / views): one JSON line
# per case with the forward / gradient verdicts.  python scripts/gpu/parity_sweep.py
import json
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import fullsize  # noqa: E402

CASES = [("c4", 0, 2), ("c1", 0, 5), ("c3", 5, 2), ("c2", 0, 3)]  # (target set: seed 1)
for cfg, view, seed in CASES:
    rep, fok, gok = fullsize.run_case(cfg, view=view, bwd=cfg != "c2", seed=seed, threads=os.cpu_count())
    print(json.dumps({"case": rep["case"], "forward_ok": fok, "grads_ok": gok,
                      "forward": rep.get("forward"), "grads": rep.get("grads")}, default=str), flush=True)
