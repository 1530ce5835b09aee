import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
    # the oracle's C restatement is test infrastructure; build it on demand
    if not os.path.exists(os.path.join(REPO, "oracle", "libraster_oracle.so")):
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def golden_scene_camera(g):
    from paper_2501_18630_b200.camera import Camera
    from paper_2501_18630_b200.scenes import SbSplatScene, SplatScene

    if "sh" in g:
        scene = SplatScene(positions=g["positions"], rotations=g["rotations"], log_scales=g["log_scales"],
                           opacity_raw=g["opacity_raw"], shapes=g["shapes"], sh=g["sh"])
    else:
        scene = SbSplatScene(positions=g["positions"], rotations=g["rotations"], log_scales=g["log_scales"],
                             opacity_raw=g["opacity_raw"], shapes=g["shapes"], base_colors=g["base_colors"],
                             lobe_axes=g["lobe_axes"], lobe_colors=g["lobe_colors"])
    fx, fy, cx, cy = g["intr"]
    w, h = (int(v) for v in g["size"])
    return scene, Camera(g["w2c"], fx, fy, cx, cy, w, h)


def toy_camera(width=32, height=32, fov=0.9, eye=(0.0, 0.0, -4.0)):
    """tests/conftest.py:9-12 of the reference."""
    from paper_2501_18630_b200.camera import Camera

    return Camera.from_lookat(eye, (0, 0, 0), (0, 1, 0), fov, width, height)


def random_scene(rng, n, degree=1, spread=0.8, scale_range=(0.05, 0.35), opacity_range=(0.2, 0.8),
                 shape_range=(-1.5, 1.5)):
    """SH analogue of the reference's random_scene (tests/conftest.py:15-31)."""
    from paper_2501_18630_b200.scenes import SplatScene

    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(*opacity_range, n)
    k = (degree + 1) ** 2
    sh = rng.normal(0.0, 0.15, (n, k, 3))
    sh[:, 0, :] = rng.uniform(0.0, 1.0, (n, 3)) / 0.28209479177387814
    return SplatScene(
        positions=rng.uniform(-spread, spread, (n, 3)).astype(np.float32),
        rotations=q.astype(np.float32),
        log_scales=np.log(rng.uniform(*scale_range, (n, 3))).astype(np.float32),
        opacity_raw=(np.log(op) - np.log1p(-op)).astype(np.float32),
        shapes=rng.uniform(*shape_range, n).astype(np.float32),
        sh=sh.astype(np.float32),
    )


def have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not have_gpu():
        pytest.skip("no CUDA device")
    import torch

    return torch.device("cuda:0")
