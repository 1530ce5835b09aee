"""Pinhole camera with the reference's conventions (host-side, fp64).

Mirrors ``betasplat.primitive.Camera`` (/root/reference/pkg/src/betasplat/primitive.py:83-137):
world->camera 4x4 with OpenCV axes (+z forward, +y down), ``fx = 0.5 W / tan(fov_x/2)``
(horizontal fov), ``fy = fx``, principal point ``((W-1)/2, (H-1)/2)`` so pixel (row i,
col j) sits at continuous coordinates (x=j, y=i).  Same validation errors (ValueError for
a non-4x4 matrix, a non-orthonormal rotation block, or an empty image).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Camera:
    world_to_camera: np.ndarray  # (4, 4) fp64
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        self.world_to_camera = np.asarray(self.world_to_camera, dtype=np.float64)
        if self.world_to_camera.shape != (4, 4):
            raise ValueError("world_to_camera must be 4x4")
        r = self.rotation
        if np.max(np.abs(r @ r.T - np.eye(3))) > 1e-6:
            raise ValueError("rotation block is not orthonormal")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be at least 1x1")
        self.width = int(self.width)
        self.height = int(self.height)

    @property
    def rotation(self) -> np.ndarray:
        return self.world_to_camera[:3, :3]

    @property
    def translation(self) -> np.ndarray:
        return self.world_to_camera[:3, 3]

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @property
    def tiles_x(self) -> int:
        return (self.width + 15) // 16

    @property
    def tiles_y(self) -> int:
        return (self.height + 15) // 16

    @classmethod
    def from_lookat(cls, eye, target, up, fov_x, width, height) -> "Camera":
        """primitive.py:123-137: rows of the rotation are (right, down, forward)."""
        eye = np.asarray(eye, dtype=np.float64)
        fwd = np.asarray(target, dtype=np.float64) - eye
        fwd = fwd / np.linalg.norm(fwd)
        right = np.cross(fwd, np.asarray(up, dtype=np.float64))
        right = right / np.linalg.norm(right)
        down = np.cross(fwd, right)
        rot = np.stack([right, down, fwd])
        w2c = np.eye(4)
        w2c[:3, :3] = rot
        w2c[:3, 3] = -rot @ eye
        f = 0.5 * width / np.tan(0.5 * fov_x)
        return cls(w2c, f, f, (width - 1) / 2.0, (height - 1) / 2.0, width, height)
