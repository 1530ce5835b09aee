"""Kernel-agnostic MCMC densification on the device (mirror of betasplat.mcmc, mcmc.py).

Same names, arguments and errors as the reference module; the work runs in libbsr
(csrc/mcmc.cu) on the flat parameter buffer and its Adam moments:

  find_dead          mcmc.py:32-36    bsr_find_dead      ordered compaction, fp64 sigmoid
  plan_relocation    mcmc.py:49-70    bsr_sample_live    opacity-weighted multinomial draw
  apply_relocation   mcmc.py:86-106   bsr_apply_relocation
  grow               mcmc.py:108-146  bsr_sample_live + bsr_grow

``rng`` is either a numpy ``Generator`` -- then the draws are numpy's own
(``rng.random(k)`` fed through ``choice``'s cdf / searchsorted rule), so a run matches the
reference draw for draw -- or a :class:`DeviceRNG`, a counter-based Philox stream on the
device that needs no host round trip.  Index arrays and per-target counts stay on the
device; ``RelocationPlan.multiplicity`` materialises the reference's dict on demand.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .primitive import PrimitiveSet, group_layout

DEAD_THRESHOLD = 0.005  # mcmc.py:25
GROWTH_RATE = 0.05  # mcmc.py:26


class AllDeadError(RuntimeError):
    """Every primitive fell below the pruning threshold (training diverged)."""


class DeviceRNG:
    """Philox4x32-10 stream on the device: (seed, offset) names every draw; each use
    advances the offset, so repeated calls never reuse a counter."""

    def __init__(self, seed: int = 0):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.offset = 0

    def advance(self, k: int = 1) -> int:
        o = self.offset
        self.offset += int(k)
        return o

    def domain(self, name: str, size: int = 1 << 40) -> int:
        """Base offset of a named counter range reserved once per stream (e.g. the
        step-keyed noise of train(), whose counters must never meet the MCMC draws')."""
        doms = self.__dict__.setdefault("_domains", {})
        if name not in doms:
            doms[name] = self.advance(size)
        return doms[name]


def _stream():
    return _lib.stream_ptr()


def _scratch(n: int, device):
    nb = ctypes.c_uint64()
    _lib.check(_lib.load().bsr_mcmc_scratch_bytes(int(n), ctypes.byref(nb)), "mcmc")
    return torch.empty(max(int(nb.value), 1), dtype=torch.uint8, device=device), int(nb.value)


def _check_threshold(threshold):
    if not 0.0 < threshold < 1.0:
        raise ValueError("threshold must lie in (0, 1)")


def find_dead(prims: PrimitiveSet, threshold: float = DEAD_THRESHOLD) -> torch.Tensor:
    """Indices (device int64, ascending) of primitives with opacity below ``threshold``."""
    _check_threshold(threshold)
    _lib.require_cuda()
    dev = prims.flat.device
    n = len(prims)
    dead = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    scratch, nb = _scratch(n, dev)
    _lib.check(_lib.load().bsr_find_dead(prims.opacity_raw.data_ptr(), n, float(threshold), dead.data_ptr(),
                                         count.data_ptr(), scratch.data_ptr(), nb, _stream()), "find_dead")
    return dead[: int(count.item())]


@dataclass
class RelocationPlan:
    """Dead-to-live assignment with per-target clone multiplicities (mcmc.py:39-46).

    ``counts[t]`` (device int32, length N) is the number of copies landing on t, so the
    reference's ``multiplicity[t] == counts[t] + 1``."""

    dead: torch.Tensor
    targets: torch.Tensor
    counts: torch.Tensor
    _mult: dict | None = field(default=None, repr=False)

    @property
    def multiplicity(self) -> dict:
        if self._mult is None:
            c = self.counts.cpu().numpy()
            nz = np.nonzero(c)[0]
            self._mult = {int(t): int(c[t]) + 1 for t in nz}
        return self._mult


def _sample(prims: PrimitiveSet, threshold, exclude, n_draw, rng, err_msg):
    """Opacity-weighted draw of ``n_draw`` live indices (live = o >= threshold minus
    ``exclude``).  Returns (indices, counts); raises AllDeadError when nothing is live."""
    dev = prims.flat.device
    n = len(prims)
    lib = _lib.load()
    scratch, nb = _scratch(n, dev)
    counts = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    live = torch.zeros(1, dtype=torch.int64, device=dev)
    out = torch.empty(max(n_draw, 1), dtype=torch.int64, device=dev)
    excl = exclude if exclude is not None and exclude.numel() else None
    ex_ptr, ex_cap = (excl.data_ptr(), excl.numel()) if excl is not None else (None, 0)

    def call(k, uniforms, seed, offset):
        _lib.check(lib.bsr_sample_live(prims.opacity_raw.data_ptr(), n, float(threshold), ex_ptr, None, ex_cap,
                                       None, k, _lib.ptr(uniforms), seed, offset, out.data_ptr(),
                                       counts.data_ptr(), live.data_ptr(), scratch.data_ptr(), nb, _stream()),
                   "sample_live")

    if isinstance(rng, DeviceRNG):
        call(n_draw, None, rng.seed, rng.advance(1))
        if int(live.item()) == 0:
            raise AllDeadError(err_msg)
    else:
        # numpy Generator: the live check comes first (the reference raises before drawing),
        # then numpy's own uniforms drive choice()'s cdf / searchsorted rule
        call(0, None, 0, 0)
        if int(live.item()) == 0:
            raise AllDeadError(err_msg)
        if n_draw > 0:
            u = torch.from_numpy(np.ascontiguousarray(rng.random(n_draw), dtype=np.float64)).to(dev)
            call(n_draw, u, 0, 0)
    return out[:n_draw], counts[:n]


def plan_relocation(prims: PrimitiveSet, dead, rng, threshold: float = DEAD_THRESHOLD) -> RelocationPlan:
    """Draw a live target for every dead primitive, odds proportional to opacity."""
    _check_threshold(threshold)
    _lib.require_cuda()
    dev = prims.flat.device
    dead = torch.as_tensor(dead, dtype=torch.int64, device=dev).reshape(-1)
    targets, counts = _sample(prims, threshold, dead, int(dead.numel()), rng,
                              f"no live primitives left ({int(dead.numel())} dead of {len(prims)})")
    return RelocationPlan(dead, targets, counts)


def new_opacity(o, n):
    """Opacity of each of ``n`` stacked copies, ``1 - (1 - o)^(1/n)`` (mcmc.py:73-83)."""
    o = np.asarray(o, dtype=np.float64)
    out = o if n == 1 else 1.0 - np.power(1.0 - o, 1.0 / n)
    return out if out.ndim else float(out)


def apply_relocation(prims: PrimitiveSet, plan: RelocationPlan, adam_state=None, floor: float = DEAD_THRESHOLD):
    """Overwrite dead primitives with their targets (opacity adjusted), in place; touched
    rows get zeroed optimizer moments."""
    d = int(plan.dead.numel())
    if d == 0:
        return prims
    _lib.require_cuda()
    dev = prims.flat.device
    count = torch.tensor([d], dtype=torch.int64, device=dev)
    lc = prims.layout_c()
    m = v = None
    if adam_state is not None:
        m, v = adam_state.exp_avg, adam_state.exp_avg_sq
    _lib.check(_lib.load().bsr_apply_relocation(
        prims.flat.data_ptr(), ctypes.byref(lc), _lib.ptr(m), _lib.ptr(v), plan.dead.data_ptr(),
        plan.targets.data_ptr(), count.data_ptr(), d, plan.counts.data_ptr(), float(floor), _stream()),
        "apply_relocation")
    return prims


def grow(prims: PrimitiveSet, budget: int, rng, adam_state=None, rate: float = GROWTH_RATE,
         dead_threshold: float = DEAD_THRESHOLD) -> PrimitiveSet:
    """Add up to ``rate`` new primitives (fraction of current) toward ``budget``; returns
    the grown set (``adam_state`` buffers are replaced by grown ones)."""
    n = len(prims)
    if budget < n:
        raise ValueError(f"budget {budget} below current count {n}")
    n_add = min(int(rate * n), budget - n)
    if n_add <= 0:
        return prims
    _lib.require_cuda()
    dev = prims.flat.device
    sources, counts = _sample(prims, dead_threshold, None, n_add, rng, "cannot grow: no live primitives")
    _, total = group_layout(n + n_add, prims.k, prims.lobes)
    # zeros, not empty: bsr_grow writes width * n floats per group and leaves the 16-byte
    # alignment padding between groups alone; Adam runs over the whole flat range
    flat = torch.zeros(total, dtype=torch.float32, device=dev)
    grown = PrimitiveSet.from_flat(n + n_add, prims.k, flat, prims.lobes)
    src_lc, dst_lc = prims.layout_c(), grown.layout_c()
    sm = sv = dm = dv = None
    if adam_state is not None:
        sm, sv = adam_state.exp_avg, adam_state.exp_avg_sq
        dm, dv = torch.zeros_like(flat), torch.zeros_like(flat)
    _lib.check(_lib.load().bsr_grow(
        prims.flat.data_ptr(), ctypes.byref(src_lc), _lib.ptr(sm), _lib.ptr(sv), flat.data_ptr(),
        ctypes.byref(dst_lc), _lib.ptr(dm), _lib.ptr(dv), sources.data_ptr(), n_add, counts.data_ptr(),
        float(dead_threshold), _stream()), "grow")
    if adam_state is not None:
        adam_state.exp_avg, adam_state.exp_avg_sq = dm, dv
    return grown


def preservation_error(shape, o, n, points=4096, kernel=None):
    """Max deviation between a primitive and its N-way opacity-split composite
    (mcmc.py:149-161; host-side diagnostic of the relocation rule)."""
    x = np.linspace(0.0, 1.0, points)
    if kernel is not None:
        f = np.asarray(kernel(x), dtype=np.float64)
    else:
        f = (1.0 - x) ** (4.0 * np.exp(np.clip(shape, -10.0, 10.0)))
    o_new = new_opacity(o, n)
    dens = o_new * f if n == 1 else 1.0 - (1.0 - o_new * f) ** n
    return float(np.max(np.abs(o * f - dens)))


__all__ = ["DEAD_THRESHOLD", "GROWTH_RATE", "AllDeadError", "DeviceRNG", "RelocationPlan", "find_dead",
           "plan_relocation", "new_opacity", "apply_relocation", "grow", "preservation_error"]
