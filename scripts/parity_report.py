"""Parity report (diagnostics, GPU box): full-size BASELINE cases and the needle scene,
printed as one JSON line per case (no asserts; tests/test_gpu_fullsize.py asserts).

    python scripts/parity_report.py c1 c2 c3 c4 needle
"""

import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import fullsize  # noqa: E402


def needle_case():
    from conftest import random_scene, toy_camera
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import PrimitiveSet, render_backward, render_tiled

    rng = np.random.default_rng(97)
    scene = random_scene(rng, 240, degree=2, spread=0.7, scale_range=(0.02, 0.1))
    k = 120
    scene.log_scales[:k] = np.log(np.array([0.8, 0.004, 0.004], np.float32))
    cam = toy_camera(256, 192)
    bg = np.ones(3)
    up = rng.standard_normal((192, 256, 3))
    fwd = orc.forward(scene, cam, bg, core="c")
    ref = orc.backward(scene, cam, bg, up, fwd, core="c")
    prims = PrimitiveSet.from_scene(scene)
    out = render_tiled(prims, cam, bg)
    g = render_backward(prims, cam, bg, up.astype(np.float32), forward_out=out)
    rep = {"case": "needles"}
    for name in fullsize.GROUPS:
        a = getattr(g, name).cpu().numpy()
        b = ref[name]
        scale = max(np.abs(b).max(), 1e-30)
        r = np.abs(a - b) / (1e-3 * np.abs(b) + 1e-5 * scale)
        rep[name] = {"needles": float(r[:k].max()), "others": float(r[k:].max())}
    return rep


def main():
    cases = sys.argv[1:] or ["needle", "c1"]
    for c in cases:
        t0 = time.perf_counter()
        try:
            if c == "needle":
                rep = needle_case()
            elif c == "sb":
                rep, fok, gok = fullsize.run_sb_case()
                rep["forward_ok"], rep["grads_ok"] = fok, gok
            else:
                cfg, _, view = c.partition(":")
                rep, fok, gok = fullsize.run_case(cfg, view=int(view or 0), bwd=cfg != "c2")
                rep["forward_ok"], rep["grads_ok"] = fok, gok
        except Exception as e:  # report and continue with the next case
            import traceback

            rep = {"case": c, "error": repr(e), "tb": traceback.format_exc()[-2000:]}
        rep["wall_s"] = round(time.perf_counter() - t0, 1)
        print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    main()
