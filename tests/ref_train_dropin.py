"""Run the REFERENCE's training loop (betasplat.training.train, training.py:313-406) twice on
its own toy dataset: once unmodified, once with its renderer switched by import to the
reference-typed B200 drop-in (paper_2501_18630_b200.compat) -- the INTEGRATION.md section 2
change.  Prints one JSON line with both runs' metrics (tests/test_gpu_reference_suite.py)."""

import json
import sys
import tempfile

import numpy as np

from betasplat import sceneio, toy, training

from paper_2501_18630_b200 import compat


def run(ds, patched):
    cfg = training.TrainConfig(total_steps=80, densify_start=30, densify_end=70, densify_interval=20,
                               max_primitives=400, init_count=300, eval_interval=40, lambda_opacity=5e-5,
                               lambda_scale=1e-4)
    orig = training.render_tiled, training.render_backward
    if patched:
        training.render_tiled, training.render_backward = compat.render_tiled, compat.render_backward
    try:
        rng = np.random.default_rng(0)
        init = sceneio.initialize_scene(ds, cfg, rng)
        res = training.train(ds, cfg, rng, initial=init)
    finally:
        training.render_tiled, training.render_backward = orig
    return {"steps": res.steps_run, "best_psnr": float(res.best_psnr), "n": len(res.primitives.positions),
            "loss": [float(m["loss"]) for m in res.metrics],
            "psnr": [float(m["psnr"]) for m in res.metrics if m["psnr"] != ""]}


def main():
    with tempfile.TemporaryDirectory() as tmp:
        toy.make_toy(tmp, preset="spheres", seed=11, views=8, size=64, count=80)
        ds = sceneio.load_transforms(tmp)
        out = {"reference": run(ds, False), "b200": run(ds, True)}
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
