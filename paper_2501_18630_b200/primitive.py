"""Device-resident primitive parameters (the reference's ``PrimitiveSet`` layout).

``PrimitiveSet`` mirrors betasplat.primitive.PrimitiveSet (primitive.py:387-494): a
struct-of-arrays of UNCONSTRAINED parameters -- opacity pre-sigmoid, scales pre-exp,
quaternions (wxyz) unnormalised -- with SH-3 colour (N, K, 3) in place of the
Spherical-Beta lobes.

B200 layout: all groups live in ONE flat fp32 CUDA buffer, group-major
    [positions 3N | rotations 4N | log_scales 3N | opacity_raw N | shapes N | sh 3KN]
so the gradient of a whole set is one contiguous buffer for the NCCL all-reduce and the
fused Adam kernel (per-group learning rates by range), and the SH block starts 16-byte
aligned for float4 loads.
"""

from __future__ import annotations

import numpy as np
import torch

GROUPS = ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh")
# reference PARAM_NAMES order (primitive.py:497-506) with SH in place of SB colour
PARAM_NAMES = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "sh")


def group_layout(n: int, k: int):
    """[(name, start, stop, shape)] of the flat buffer."""
    widths = {"positions": 3, "rotations": 4, "log_scales": 3, "opacity_raw": 1, "shapes": 1, "sh": 3 * k}
    shapes = {"positions": (n, 3), "rotations": (n, 4), "log_scales": (n, 3), "opacity_raw": (n,),
              "shapes": (n,), "sh": (n, k, 3)}
    out, off = [], 0
    for g in GROUPS:
        out.append((g, off, off + widths[g] * n, shapes[g]))
        off += widths[g] * n
        off = (off + 3) // 4 * 4  # every group starts 16-byte aligned (float4 access)
    return out, off


class FlatGroups:
    """A flat fp32 buffer with named group views (shared by PrimitiveSet / GradientBuffer)."""

    def __init__(self, n: int, k: int, flat: torch.Tensor):
        self.n, self.k = int(n), int(k)
        self.layout, total = group_layout(self.n, self.k)
        if flat.numel() != total or flat.dtype != torch.float32 or not flat.is_contiguous():
            raise ValueError("flat buffer has the wrong size / dtype")
        self.flat = flat
        for name, a, b, shape in self.layout:
            setattr(self, name, flat[a:b].view(shape))

    def __len__(self):
        return self.n

    @property
    def sh_coeffs(self) -> int:
        return self.k

    def parameters(self) -> dict:
        return {name: getattr(self, name) for name in PARAM_NAMES}

    def group_ends(self):
        return [b for _, _, b, _ in self.layout]


class PrimitiveSet(FlatGroups):
    def __init__(self, positions, rotations, log_scales, opacity_raw, shapes, sh, device="cuda"):
        arrs = dict(positions=positions, rotations=rotations, log_scales=log_scales,
                    opacity_raw=opacity_raw, shapes=shapes, sh=sh)
        n = int(np.asarray(positions.shape)[0])
        sh_shape = tuple(sh.shape)
        if len(sh_shape) != 3 or sh_shape[2] != 3 or sh_shape[1] not in (1, 4, 9, 16):
            raise ValueError("sh must be (N, K, 3) with K in {1, 4, 9, 16}")
        k = sh_shape[1]
        for name, a in arrs.items():
            if tuple(a.shape)[0] != n:
                raise ValueError(f"{name} row count mismatch")
        _, total = group_layout(n, k)
        flat = torch.zeros(total, dtype=torch.float32, device=device)
        super().__init__(n, k, flat)
        for name, a in arrs.items():
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            getattr(self, name).copy_(t.to(dtype=torch.float32).reshape(getattr(self, name).shape))

    @classmethod
    def from_scene(cls, scene, device="cuda") -> "PrimitiveSet":
        return cls(scene.positions, scene.rotations, scene.log_scales, scene.opacity_raw, scene.shapes,
                   scene.sh, device=device)

    @classmethod
    def from_flat(cls, n, k, flat) -> "PrimitiveSet":
        obj = cls.__new__(cls)
        FlatGroups.__init__(obj, n, k, flat)
        return obj

    @property
    def opacities(self):
        return torch.sigmoid(self.opacity_raw)

    @property
    def scales(self):
        return torch.exp(self.log_scales)

    def copy(self) -> "PrimitiveSet":
        return PrimitiveSet.from_flat(self.n, self.k, self.flat.clone())

    def take(self, idx) -> "PrimitiveSet":
        idx = torch.as_tensor(idx, device=self.flat.device, dtype=torch.long)
        return PrimitiveSet(*(getattr(self, g)[idx] for g in GROUPS), device=self.flat.device)

    def to_numpy(self) -> dict:
        return {g: getattr(self, g).detach().cpu().numpy() for g in GROUPS}


class GradientBuffer(FlatGroups):
    """Per-parameter gradients aligned with the primitive set (rasterizer.py:49-80)."""

    def __init__(self, n, k, flat=None, device="cuda"):
        _, total = group_layout(n, k)
        if flat is None:
            flat = torch.zeros(total, dtype=torch.float32, device=device)
        super().__init__(n, k, flat)
        self.screen_grad_norm = torch.zeros(n, dtype=torch.float32, device=flat.device)

    @classmethod
    def zeros_for(cls, prims: PrimitiveSet) -> "GradientBuffer":
        return cls(prims.n, prims.k, device=prims.flat.device)

    def zero_(self):
        self.flat.zero_()
        self.screen_grad_norm.zero_()
        return self
