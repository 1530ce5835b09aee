"""Seeded synthetic workloads for the BASELINE.json configs (c0..c4).

No public dataset is named by BASELINE.json and the paper's scenes are not available
offline, so these generators stand in for them.  Every array is
drawn in fp64 from ONE ``np.random.default_rng(seed)`` stream in a fixed order

    means, log-scales, quaternions, opacity logits, SH DC, SH rest

and rounded to fp32, so the GPU path and the fp64 oracle consume identical values.
``shapes`` are 0 (Beta exponent 4, the reference's "Gaussian-like" kernel, kernel.py:42-44).
SH layout is (N, K, 3) with the DC row first (appearance.py:212-232).
Cameras use the reference convention: horizontal fov, world up +y (toy.py:129-139);
"upper hemisphere" = y > 0, rejecting y > 0.99 where ``from_lookat`` degenerates.
Hemisphere cameras come from their own stream (``camera_rng(seed)``), so a workload's
cameras do not depend on its primitive count: a reduced-size parity case, the bench's
GPU arm and its CPU baseline all see the same views.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .camera import Camera

PARAM_ORDER = ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh")


@dataclass
class SplatScene:
    """SoA primitive parameters (unconstrained, like ``PrimitiveSet``, primitive.py:387-426)."""

    positions: np.ndarray  # (N, 3)
    rotations: np.ndarray  # (N, 4) wxyz, unnormalised
    log_scales: np.ndarray  # (N, 3)
    opacity_raw: np.ndarray  # (N,) pre-sigmoid
    shapes: np.ndarray  # (N,) Beta shape b
    sh: np.ndarray  # (N, K, 3)

    def __len__(self):
        return int(self.positions.shape[0])

    @property
    def sh_degree(self) -> int:
        return int(round(np.sqrt(self.sh.shape[1]))) - 1

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in PARAM_ORDER}

    def astype(self, dtype) -> "SplatScene":
        return SplatScene(**{k: np.ascontiguousarray(v, dtype=dtype) for k, v in self.arrays().items()})

    def take(self, idx) -> "SplatScene":
        return SplatScene(**{k: v[idx].copy() for k, v in self.arrays().items()})


@dataclass
class SbSplatScene:
    """SoA parameters with the reference's Spherical-Beta colour (primitive.py:387-426)."""

    positions: np.ndarray  # (N, 3)
    rotations: np.ndarray  # (N, 4)
    log_scales: np.ndarray  # (N, 3)
    opacity_raw: np.ndarray  # (N,)
    shapes: np.ndarray  # (N,)
    base_colors: np.ndarray  # (N, 3)
    lobe_axes: np.ndarray  # (N, M, 3)
    lobe_colors: np.ndarray  # (N, M, 3)

    def __len__(self):
        return int(self.positions.shape[0])

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes",
                                             "base_colors", "lobe_axes", "lobe_colors")}

    def astype(self, dtype) -> "SbSplatScene":
        return SbSplatScene(**{k: np.ascontiguousarray(v, dtype=dtype) for k, v in self.arrays().items()})

    def take(self, idx) -> "SbSplatScene":
        return SbSplatScene(**{k: v[idx].copy() for k, v in self.arrays().items()})


def fibonacci_directions(m):
    """appearance.py:29-37: m quasi-uniform unit directions."""
    if m == 0:
        return np.zeros((0, 3))
    i = np.arange(m) + 0.5
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    z = 1.0 - 2.0 * i / m
    rho = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    return np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=-1)


def sb_random_scene(rng, n, lobes=2, spread=0.8, scale_range=(0.05, 0.35), opacity_range=(0.2, 0.8),
                    lobe_color_scale=0.3) -> SbSplatScene:
    """The reference tests' random scene generator (tests/conftest.py:15-31), fp32-rounded."""
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    axes = fibonacci_directions(lobes)[None] * np.exp(rng.uniform(-0.3, 0.8, (n, lobes, 1)))
    op = rng.uniform(*opacity_range, n)
    f = np.float32
    return SbSplatScene(
        positions=rng.uniform(-spread, spread, (n, 3)).astype(f),
        opacity_raw=(np.log(op) - np.log1p(-op)).astype(f),
        rotations=q.astype(f),
        log_scales=np.log(rng.uniform(*scale_range, (n, 3))).astype(f),
        shapes=rng.uniform(-1.5, 1.5, n).astype(f),
        base_colors=rng.uniform(0.0, 1.0, (n, 3)).astype(f),
        lobe_axes=axes.astype(f),
        lobe_colors=(rng.uniform(-0.2, 1.0, (n, lobes, 3)) * lobe_color_scale).astype(f),
    )


@dataclass
class Workload:
    name: str
    scene: SplatScene
    cameras: list = field(default_factory=list)
    background: np.ndarray = field(default_factory=lambda: np.ones(3))
    train: bool = False
    target_seed: int | None = None


def _quats(rng, n):
    q = rng.standard_normal((n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _sh(rng, n, degree, dc_std, rest_std):
    k = (degree + 1) ** 2
    sh = np.empty((n, k, 3))
    sh[:, 0, :] = rng.normal(0.0, dc_std, (n, 3))
    if k > 1:
        sh[:, 1:, :] = rng.normal(0.0, rest_std, (n, k - 1, 3))
    return sh


def _finish(pos, logs, quat, logit, sh) -> SplatScene:
    n = pos.shape[0]
    f = np.float32
    return SplatScene(
        positions=np.ascontiguousarray(pos, dtype=f),
        rotations=np.ascontiguousarray(quat, dtype=f),
        log_scales=np.ascontiguousarray(logs, dtype=f),
        opacity_raw=np.ascontiguousarray(logit, dtype=f),
        shapes=np.zeros(n, dtype=f),
        sh=np.ascontiguousarray(sh, dtype=f),
    )


def hemisphere_eye(rng, radius):
    while True:
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        d[1] = abs(d[1])
        if d[1] <= 0.99:
            return radius * d


def camera_rng(seed):
    """The cameras' stream, independent of the scene arrays (and of N)."""
    return np.random.default_rng([int(seed), 0x63616D])


def scene_c0(seed=0, n=10_000):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1.0, 1.0, (n, 3))
    logs = rng.normal(-4.0, 0.5, (n, 3))
    quat = _quats(rng, n)
    logit = rng.normal(0.0, 1.0, n)
    sh = _sh(rng, n, 0, 0.5, 0.0)
    return _finish(pos, logs, quat, logit, sh), rng


def scene_c1(seed=0, n=100_000):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1.0, 1.0, (n, 3))
    logs = rng.normal(-4.0, 0.5, (n, 3))
    quat = _quats(rng, n)
    logit = rng.normal(0.0, 1.0, n)
    sh = _sh(rng, n, 3, 0.5, 0.05)
    return _finish(pos, logs, quat, logit, sh), rng


def scene_c2(seed=0, n=1_000_000):
    rng = np.random.default_rng(seed)
    pos = np.clip(rng.normal(0.0, 2.0, (n, 3)), -6.0, 6.0)
    logs = rng.normal(-5.0, 0.7, (n, 3))
    quat = _quats(rng, n)
    logit = rng.normal(0.0, 1.5, n)
    sh = _sh(rng, n, 3, 0.5, 0.05)
    return _finish(pos, logs, quat, logit, sh), rng


def scene_c4(seed=0, n=6_000_000):
    rng = np.random.default_rng(seed)
    n_dense = int(round(0.7 * n))
    pos = np.concatenate([rng.normal(0.0, 0.5, (n_dense, 3)), rng.uniform(-10.0, 10.0, (n - n_dense, 3))])
    logs = rng.normal(-5.5, 1.0, (n, 3))
    quat = _quats(rng, n)
    logit = rng.normal(1.0, 1.0, n)
    sh = _sh(rng, n, 3, 0.5, 0.05)
    return _finish(pos, logs, quat, logit, sh), rng


def make_workload(name: str, seed: int = 0, n: int | None = None, views: int | None = None,
                  width: int | None = None, height: int | None = None) -> Workload:
    """Build a BASELINE config (``c0``..``c4``); ``n``/``views``/size override for tests."""
    up = (0.0, 1.0, 0.0)
    if name == "c0":
        scene, _ = scene_c0(seed, n or 10_000)
        w, h = width or 256, height or 256
        cams = [Camera.from_lookat((0, 0, 4), (0, 0, 0), up, np.deg2rad(60.0), w, h)]
        return Workload(name, scene, cams)
    if name == "c1":
        scene, _ = scene_c1(seed, n or 100_000)
        w, h = width or 800, height or 800
        cams = [Camera.from_lookat((0, 0, 4), (0, 0, 0), up, np.deg2rad(60.0), w, h)]
        return Workload(name, scene, cams, train=True, target_seed=seed + 1)
    if name == "c2":
        scene, _ = scene_c2(seed, n or 1_000_000)
        rng = camera_rng(seed)
        w, h = width or 1920, height or 1080
        cams = [Camera.from_lookat(hemisphere_eye(rng, 8.0), (0, 0, 0), up, np.deg2rad(50.0), w, h)]
        return Workload(name, scene, cams)
    if name == "c3":
        scene, _ = scene_c2(seed, n or 3_000_000)
        rng = camera_rng(seed)
        w, h = width or 1600, height or 1067
        cams = [Camera.from_lookat(hemisphere_eye(rng, 8.0), (0, 0, 0), up, np.deg2rad(50.0), w, h)
                for _ in range(views or 32)]
        return Workload(name, scene, cams, train=True, target_seed=seed + 1)
    if name == "c4":
        scene, _ = scene_c4(seed, n or 6_000_000)
        rng = camera_rng(seed)
        w, h = width or 3840, height or 2160
        cams = [Camera.from_lookat(hemisphere_eye(rng, 3.0), (0, 0, 0), up, np.deg2rad(70.0), w, h)]
        return Workload(name, scene, cams, train=True, target_seed=None)
    raise ValueError(f"unknown workload {name!r} (expected c0..c4)")


def target_scene(name: str, seed: int, n: int | None = None) -> SplatScene:
    """The second seeded Gaussian set of the same distribution (configs 1 and 3)."""
    gen = {"c0": scene_c0, "c1": scene_c1, "c2": scene_c2, "c3": scene_c2, "c4": scene_c4}[name]
    default_n = {"c0": 10_000, "c1": 100_000, "c2": 1_000_000, "c3": 3_000_000, "c4": 6_000_000}[name]
    return gen(seed, n or default_n)[0]
