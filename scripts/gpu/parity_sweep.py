# Extra full-size parity cases beyond the pytest suite (other seeds / views): one JSON line
# per case with the forward / gradient verdicts.  python scripts/gpu/parity_sweep.py
import json
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import fullsize  # noqa: E402

CASES = [("c4", 0, 2), ("c1", 0, 5), ("c3", 5, 2), ("c2", 0, 3)]  # (target set: seed 1)
if len(sys.argv) > 1 and sys.argv[1] == "wide":  # the round's wider sweep
    CASES = [("c4", 0, 1), ("c4", 0, 3), ("c3", 3, 0), ("c3", 9, 1), ("c3", 25, 3), ("c1", 0, 1), ("c1", 0, 2),
             ("c1", 0, 3), ("c2", 0, 1), ("c2", 0, 2), ("c2", 0, 4)]
for cfg, view, seed in CASES:
    rep, fok, gok = fullsize.run_case(cfg, view=view, bwd=cfg != "c2", seed=seed, threads=os.cpu_count())
    print(json.dumps({"case": rep["case"], "forward_ok": fok, "grads_ok": gok,
                      "forward": rep.get("forward"), "grads": rep.get("grads")}, default=str), flush=True)
