"""Reference-typed drop-in of the renderer entry points (numpy in, numpy out).

    render_tiled(prims, camera, background, threads=None, core=None)           -> RenderOutput
    render_backward(prims, camera, background, d_color, forward_out=None,
                    threads=None, core=None)                                    -> GradientBuffer
    render_masked(prims, camera, background, predicate, threads=None)           -> RenderOutput

take exactly what betasplat.rasterizer's functions take (rasterizer.py:194-321): the
reference's numpy ``PrimitiveSet`` (Spherical-Beta colour, the reference's default; or an
SH set such as scenes.SplatScene) and its ``Camera`` (any object with world_to_camera,
fx, fy, cx, cy, width, height), and return the reference's own ``RenderOutput`` /
``GradientBuffer`` types when betasplat is importable (identically-named dataclasses
otherwise), fp64 numpy arrays, contributions int64 -- so the reference's call sites
(training.train, evaluate_psnr, cli render) switch by import.

Every call runs the whole path on the device (libbsr.so); the parameters are rounded to
fp32 on upload (the north star's compute precision).  ``threads`` is accepted and
ignored; ``core`` must be None / "cuda" (the reference's core plugin seam is
``backend.get_core("cuda")``).  The reference's render_backward recomputes the forward
when ``forward_out`` is a numpy RenderOutput (rasterizer.py:243-251); so does this one,
unless ``forward_out`` came from this module (it then carries the saved device frame).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import rasterizer as _rz
from .primitive import PrimitiveSet


@dataclass
class RenderOutput:
    """betasplat.rasterizer.RenderOutput (rasterizer.py:40-46) when betasplat is absent."""

    color: np.ndarray
    alpha: np.ndarray
    contributions: np.ndarray
    raw_color: np.ndarray
    transmittance: np.ndarray


@dataclass
class GradientBuffer:
    """betasplat.rasterizer.GradientBuffer (rasterizer.py:49-80) field set, plus ``sh`` for
    SH-colour sets."""

    positions: np.ndarray
    opacity_raw: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    shapes: np.ndarray
    base_colors: np.ndarray | None = None
    lobe_axes: np.ndarray | None = None
    lobe_colors: np.ndarray | None = None
    screen_grad_norm: np.ndarray | None = None
    sh: np.ndarray | None = None

    def parameters(self):
        names = ("positions", "opacity_raw", "rotations", "log_scales", "shapes")
        names += ("sh",) if self.sh is not None else ("base_colors", "lobe_axes", "lobe_colors")
        return {k: getattr(self, k) for k in names}


def _ref_types():
    try:
        from betasplat import rasterizer as ref_rz  # the reference package, when installed

        return ref_rz.RenderOutput, ref_rz.GradientBuffer
    except Exception:
        return RenderOutput, GradientBuffer


def _is_sh(prims) -> bool:
    return getattr(prims, "sh", None) is not None


def to_device(prims) -> PrimitiveSet:
    """A numpy primitive set (reference SB, or SH with an ``sh`` (N, K, 3) array) on the device."""
    if isinstance(prims, PrimitiveSet):
        return prims
    if _is_sh(prims):
        return PrimitiveSet.from_scene(prims)
    return PrimitiveSet.from_reference(prims)


def _np(t, dtype=np.float64):
    return t.detach().to(torch.float64 if dtype == np.float64 else t.dtype).cpu().numpy().astype(dtype, copy=False)


class _DeviceForward:
    """Attached to a returned RenderOutput: the device output whose frame render_backward reuses."""

    __slots__ = ("out", "dev_prims")

    def __init__(self, out, dev_prims):
        self.out, self.dev_prims = out, dev_prims


def _check_core(core):
    if core not in (None, "cuda", "auto") and getattr(core, "__name__", "").rsplit(".", 1)[-1] != "cuda_core":
        raise ValueError(f"unknown backend {core!r} (this drop-in runs the 'cuda' path)")


def render_tiled(prims, camera, background, threads=None, core=None):
    """rasterizer.py:194-211 with reference types, on the B200."""
    _check_core(core)
    RO, _ = _ref_types()
    dev = to_device(prims)
    out = _rz.render_tiled(dev, camera, background, sync=True)
    trans = _np(out.transmittance)
    # alpha = 1 - T in fp64, as the reference core returns it (_raster.pyx:152)
    res = RO(color=_np(out.color), alpha=1.0 - trans, contributions=_np(out.contributions, np.int64),
             raw_color=_np(out.raw_color), transmittance=trans)
    try:
        res._b200 = _DeviceForward(out, dev)  # dataclass instances accept extra attributes
    except AttributeError:
        pass
    return res


def render_masked(prims, camera, background, predicate, threads=None):
    """rasterizer.py:214-227 with reference types."""
    mask = np.asarray(predicate(np.asarray(prims.shapes)), dtype=bool)
    keep = np.nonzero(mask)[0]
    out = render_tiled(prims.take(keep), camera, background, threads)
    contributions = np.zeros(len(prims.positions), dtype=np.int64)
    contributions[keep] = out.contributions
    out.contributions = contributions
    return out


def render_backward(prims, camera, background, d_color, forward_out=None, threads=None, core=None):
    """rasterizer.py:230-321 with reference types: exact analytic gradients of the image."""
    _check_core(core)
    _, GB = _ref_types()
    saved = getattr(forward_out, "_b200", None)
    if saved is not None:
        dev, out = saved.dev_prims, saved.out
    else:
        dev = to_device(prims)
        out = _rz.render_tiled(dev, camera, background, sync=True)
    d = np.asarray(d_color, dtype=np.float32)
    g = _rz.render_backward(dev, camera, background, d, forward_out=out)
    fields = dict(positions=_np(g.positions), opacity_raw=_np(g.opacity_raw), rotations=_np(g.rotations),
                  log_scales=_np(g.log_scales), shapes=_np(g.shapes), screen_grad_norm=_np(g.screen_grad_norm))
    if dev.color_model == "sh":
        return GradientBuffer(sh=_np(g.sh), **fields)
    fields.update(base_colors=_np(g.base_colors), lobe_axes=_np(g.lobe_axes), lobe_colors=_np(g.lobe_colors))
    return GB(**fields)
