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

import functools

import numpy as np
import torch

GEOMETRY = ("positions", "rotations", "log_scales", "opacity_raw", "shapes")
GROUPS = GEOMETRY + ("sh",)  # SH colour model (BASELINE configs)
SB_GROUPS = GEOMETRY + ("base_colors", "lobe_axes", "lobe_colors")  # Spherical Beta (reference default)
# reference PARAM_NAMES order (primitive.py:497-506); SH replaces the SB colour groups
PARAM_NAMES = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "sh")
SB_PARAM_NAMES = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "base_colors",
                  "lobe_axes", "lobe_colors")
MAX_LOBES = 4  # BSR_MAX_LOBES (include/bsr.h)


def group_widths(k: int | None = None, lobes: int | None = None) -> dict:
    """Floats per primitive of every group."""
    w = {"positions": 3, "rotations": 4, "log_scales": 3, "opacity_raw": 1, "shapes": 1}
    if lobes is None:
        w["sh"] = 3 * k
    else:
        w.update(base_colors=3, lobe_axes=3 * lobes, lobe_colors=3 * lobes)
    return w


@functools.lru_cache(maxsize=256)
def group_layout(n: int, k: int | None = None, lobes: int | None = None):
    """((name, start, stop, shape), ...) of the flat buffer for the SH (k) or SB (lobes)
    model, and its length (cached: every buffer of a set rebuilds its views from it)."""
    widths = {"positions": 3, "rotations": 4, "log_scales": 3, "opacity_raw": 1, "shapes": 1}
    shapes = {"positions": (n, 3), "rotations": (n, 4), "log_scales": (n, 3), "opacity_raw": (n,),
              "shapes": (n,)}
    if lobes is None:
        groups = GROUPS
        widths["sh"] = 3 * k
        shapes["sh"] = (n, k, 3)
    else:
        groups = SB_GROUPS
        widths.update(base_colors=3, lobe_axes=3 * lobes, lobe_colors=3 * lobes)
        shapes.update(base_colors=(n, 3), lobe_axes=(n, lobes, 3), lobe_colors=(n, lobes, 3))
    out, off = [], 0
    for g in groups:
        out.append((g, off, off + widths[g] * n, shapes[g]))
        off += widths[g] * n
        off = (off + 3) // 4 * 4  # every group starts 16-byte aligned (float4 access)
    return tuple(out), off


class FlatGroups:
    """A flat fp32 buffer with named group views (shared by PrimitiveSet / GradientBuffer)."""

    def __init__(self, n: int, k: int | None, flat: torch.Tensor, lobes: int | None = None):
        self.n = int(n)
        self.k = None if k is None else int(k)
        self.lobes = None if lobes is None else int(lobes)
        self.color_model = "sh" if lobes is None else "sb"
        self.layout, total = group_layout(self.n, self.k, self.lobes)
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

    @property
    def param_names(self):
        return PARAM_NAMES if self.color_model == "sh" else SB_PARAM_NAMES

    @property
    def groups(self):
        return [g for g, *_ in self.layout]

    def parameters(self) -> dict:
        return {name: getattr(self, name) for name in self.param_names}

    def group_ends(self):
        return [b for _, _, b, _ in self.layout]

    def layout_c(self):
        """The group table as the C-ABI's bsr_layout (include/bsr.h)."""
        from . import _lib

        lc = _lib.LayoutC()
        lc.n = self.n
        lc.n_groups = len(self.layout)
        widths = group_widths(self.k, self.lobes)
        for g, (name, a, _, _) in enumerate(self.layout):
            lc.width[g] = widths[name]
            lc.start[g] = a
        names = self.groups
        lc.g_positions, lc.g_rotations = names.index("positions"), names.index("rotations")
        lc.g_log_scales, lc.g_opacity = names.index("log_scales"), names.index("opacity_raw")
        return lc


class PrimitiveSet(FlatGroups):
    """Either SH colour (``sh`` (N,K,3)) or the reference's Spherical-Beta colour
    (``base_colors`` (N,3), ``lobe_axes`` / ``lobe_colors`` (N,M,3))."""

    def __init__(self, positions, rotations, log_scales, opacity_raw, shapes, sh=None, device="cuda",
                 base_colors=None, lobe_axes=None, lobe_colors=None):
        arrs = dict(positions=positions, rotations=rotations, log_scales=log_scales,
                    opacity_raw=opacity_raw, shapes=shapes)
        n = int(np.asarray(positions.shape)[0])
        k = lobes = None
        if sh is not None:
            sh_shape = tuple(sh.shape)
            if len(sh_shape) != 3 or sh_shape[2] != 3 or sh_shape[1] not in (1, 4, 9, 16):
                raise ValueError("sh must be (N, K, 3) with K in {1, 4, 9, 16}")
            k = sh_shape[1]
            arrs["sh"] = sh
        else:
            if base_colors is None:
                raise ValueError("need sh (SH colour) or base_colors/lobe_axes/lobe_colors (SB colour)")
            if lobe_axes is None:
                lobe_axes = np.zeros((n, 0, 3), np.float32)
                lobe_colors = np.zeros((n, 0, 3), np.float32)
            if tuple(lobe_axes.shape) != tuple(lobe_colors.shape) or len(lobe_axes.shape) != 3:
                raise ValueError("lobe_axes and lobe_colors must have matching (N, M, 3) shapes")
            lobes = int(lobe_axes.shape[1])
            if lobes > MAX_LOBES:
                raise ValueError(f"at most {MAX_LOBES} Spherical Beta lobes are supported")
            arrs.update(base_colors=base_colors, lobe_axes=lobe_axes, lobe_colors=lobe_colors)
        for name, a in arrs.items():
            if tuple(a.shape)[0] != n:
                raise ValueError(f"{name} row count mismatch")
        _, total = group_layout(n, k, lobes)
        flat = torch.zeros(total, dtype=torch.float32, device=device)
        super().__init__(n, k, flat, lobes)
        for name, a in arrs.items():
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            getattr(self, name).copy_(t.to(dtype=torch.float32).reshape(getattr(self, name).shape))

    @classmethod
    def from_scene(cls, scene, device="cuda") -> "PrimitiveSet":
        return cls(scene.positions, scene.rotations, scene.log_scales, scene.opacity_raw, scene.shapes,
                   scene.sh, device=device)

    @classmethod
    def from_reference(cls, prims, device="cuda") -> "PrimitiveSet":
        """A reference ``betasplat.PrimitiveSet`` (fp64 numpy, Spherical-Beta colour) on the
        device in fp32 -- the drop-in path for reference checkpoints."""
        return cls(prims.positions, prims.rotations, prims.log_scales, prims.opacity_raw, prims.shapes,
                   device=device, base_colors=prims.base_colors, lobe_axes=prims.lobe_axes,
                   lobe_colors=prims.lobe_colors)

    @classmethod
    def from_flat(cls, n, k, flat, lobes=None) -> "PrimitiveSet":
        obj = cls.__new__(cls)
        FlatGroups.__init__(obj, n, k, flat, lobes)
        return obj

    @property
    def opacities(self):
        return torch.sigmoid(self.opacity_raw)

    @property
    def scales(self):
        return torch.exp(self.log_scales)

    def copy(self) -> "PrimitiveSet":
        return PrimitiveSet.from_flat(self.n, self.k, self.flat.clone(), self.lobes)

    def take(self, idx) -> "PrimitiveSet":
        idx = torch.as_tensor(idx, device=self.flat.device, dtype=torch.long)
        sub = {g: getattr(self, g)[idx] for g in self.groups}
        return PrimitiveSet(**sub, device=self.flat.device)

    def to_numpy(self) -> dict:
        return {g: getattr(self, g).detach().cpu().numpy() for g in self.groups}


# GradientBuffer attributes that never depend on pending colour chains
_GRAD_META = frozenset(("n", "k", "lobes", "color_model", "layout", "groups", "param_names", "sh_coeffs",
                        "group_ends", "layout_c", "flush_pending"))


class GradientBuffer(FlatGroups):
    """Per-parameter gradients aligned with the primitive set (rasterizer.py:49-80).

    A buffer that rasterizer.render_backward accumulates several views of an SH set into
    may hold those views' colour chains deferred (``_pending``: their d rgb rows, applied
    by one bsr_color_grad_views); reading any gradient attribute applies them first, so
    the values seen are always the complete sums."""

    def __getattribute__(self, name):
        if name[:1] != "_" and name not in _GRAD_META:
            d = object.__getattribute__(self, "__dict__")
            p = d.get("_pending")
            if p is not None:
                d["_pending"] = None
                p.apply(self)
        return object.__getattribute__(self, name)

    def flush_pending(self):
        """Apply deferred colour chains now (otherwise done on the next attribute read)."""
        d = self.__dict__
        p = d.get("_pending")
        if p is not None:
            d["_pending"] = None
            p.apply(self)
        return self

    def __init__(self, n, k, flat=None, device="cuda", lobes=None):
        _, total = group_layout(n, k, lobes)
        if flat is None:
            flat = torch.zeros(total, dtype=torch.float32, device=device)
        super().__init__(n, k, flat, lobes)
        self.screen_grad_norm = torch.zeros(n, dtype=torch.float32, device=flat.device)

    @classmethod
    def zeros_for(cls, prims: PrimitiveSet) -> "GradientBuffer":
        return cls(prims.n, prims.k, device=prims.flat.device, lobes=prims.lobes)

    @classmethod
    def empty_for(cls, prims: PrimitiveSet) -> "GradientBuffer":
        """Uninitialised group rows (for a backward in overwrite mode, which writes every
        row); only the alignment padding between groups is zeroed."""
        layout, total = group_layout(prims.n, prims.k, prims.lobes)
        flat = torch.empty(total, dtype=torch.float32, device=prims.flat.device)
        prev = 0
        for _, a, b, _ in layout:
            if a > prev:
                flat[prev:a].zero_()
            prev = b
        if total > prev:
            flat[prev:total].zero_()
        return cls(prims.n, prims.k, flat=flat, lobes=prims.lobes)

    def zero_(self):
        self.flat.zero_()
        self.screen_grad_norm.zero_()
        return self
