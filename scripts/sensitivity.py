"""Conditioning of the reference gradients (diagnostics, GPU box CPU): how far the oracle's
own gradient moves when a per-record input of the raster (colour, opacity, mean, conic) is
rounded to fp32 -- the precision the device records carry.  Rows whose reference gradient
moves by more than the parity tolerance under such a rounding are ill-posed at fp32.

    python scripts/sensitivity.py c4 [rows...]
"""

import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import fullsize  # noqa: E402


def main():
    from oracle import pipeline as orc
    from paper_2501_18630_b200.scenes import make_workload

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    rows = [int(r) for r in sys.argv[2:]]
    wl = make_workload(cfg, seed=0)
    scene, cam, bg = wl.scene, wl.cameras[0], wl.background
    ref = orc.forward(scene, cam, bg, core="c")
    rng = np.random.default_rng(5)
    up = rng.standard_normal(ref["raw"].shape) * 1e-7  # upstream of the loss-gradient scale
    up[np.abs(ref["raw"]) < fullsize.KINK] = 0.0
    base = orc.backward(scene, cam, bg, up, ref, core="c")
    for keys in (["colors"], ["opac"], ["means"], ["conics"]):
        f2 = dict(ref)
        sh = dict(ref["shaded"])
        s = dict(sh["sorted"])
        for k in keys:
            s[k] = s[k].astype(np.float32).astype(np.float64)
        sh["sorted"] = s
        f2["shaded"] = sh
        g = orc.backward(scene, cam, bg, up, f2, core="c")
        rep = {"rounded": keys}
        for name in ("positions", "rotations", "log_scales"):
            r = fullsize.grad_ratio(g[name], base[name])
            rr = r.reshape(r.shape[0], -1).max(axis=1)
            rep[name] = {"max": float(rr.max()), "n_over_1": int((rr > 1).sum()),
                         "worst": [int(i) for i in np.argsort(-rr)[:4]],
                         "rows": {str(i): float(rr[i]) for i in rows}}
        print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    main()
