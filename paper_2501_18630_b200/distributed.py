"""View-batch data parallelism (config 3): one process per GPU, Gaussians replicated.

The reference trains one view per step on one process (training.py:351-361; multi-view
batches are a spec non-goal) and has no collectives.  Here a batch of
camera views is partitioned across ranks (contiguous groups of n_views / world), every
rank accumulates its views' per-Gaussian gradients into ONE flat buffer
(primitive.GradientBuffer), and the one exchange step is a sum all-reduce of that buffer
(NCCL over NVLink 5 / NVSwitch on the B200 box; gloo in the CPU tests) before the
identical Adam update on every rank.  Timings are reduced as max over ranks.
"""

from __future__ import annotations

import os

import numpy as np
import torch


def init(backend: str | None = None):
    """Initialise torch.distributed from the torchrun environment (RANK / WORLD_SIZE /
    LOCAL_RANK / MASTER_*).  Returns (rank, world, local_rank); single process -> (0, 1, 0)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not torch.distributed.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def partition_views(n_views: int, world: int, rank: int) -> range:
    """Contiguous share of the view batch for ``rank`` (remainder to the first ranks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def allreduce_grads(flat: torch.Tensor, group=None, average: bool = False) -> torch.Tensor:
    """Sum (or mean) the flat per-Gaussian gradient buffer across ranks, in place."""
    if torch.distributed.is_available() and torch.distributed.is_initialized() and \
            torch.distributed.get_world_size(group) > 1:
        torch.distributed.all_reduce(flat, op=torch.distributed.ReduceOp.SUM, group=group)
        if average:
            flat /= torch.distributed.get_world_size(group)
    return flat


def _reduce_scalar(x: float, op) -> float:
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return float(x)
    dev = "cuda" if torch.distributed.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float) -> float:
    return _reduce_scalar(x, torch.distributed.ReduceOp.MAX if torch.distributed.is_available() else None)


def sum_over_ranks(x: float) -> float:
    return _reduce_scalar(x, torch.distributed.ReduceOp.SUM if torch.distributed.is_available() else None)


def orbit_cameras(n: int, radius: float = 4.0, fov_deg: float = 60.0, width: int = 800, height: int = 800):
    """Cameras on a y-orbit around the origin (view 0 is the config-1 camera on +z)."""
    from .camera import Camera

    cams = []
    for k in range(n):
        ang = 2 * np.pi * k / max(n, 1)
        eye = (radius * np.sin(ang), 0.0, radius * np.cos(ang))
        cams.append(Camera.from_lookat(eye, (0, 0, 0), (0, 1, 0), np.deg2rad(fov_deg), width, height))
    return cams


# ----------------------------------------------------------------------------- sharded step
class ShardedOptimizer:
    """Reduce-scatter -> sharded Adam -> all-gather (SURVEY 8(e) option 2) for view-batch DP.

    The flat parameter and gradient buffers are re-homed into buffers padded to a multiple
    of 4 * world floats; rank r owns the contiguous shard [r S, (r + 1) S), S = padded / world
    (16-byte aligned, so the fused Adam kernel keeps its float4 path).  Per step:

      reduce_scatter(sum) of the gradient buffer  -> this rank's shard of the summed gradient
      fused Adam on the shard only                 (1/world of the optimiser work and state)
      all_gather of the parameter shards           -> every rank's full, identical parameters

    The bytes on the wire equal one all-reduce (2 (W-1)/W x the buffer); the Adam moments
    shrink to 1/world per rank.  The group learning rates follow the global layout: the
    kernel gets the group ends shifted by the shard offset (groups before the shard are
    empty).  Backends without reduce_scatter / all_gather on device tensors (gloo on CUDA)
    fall back to all_reduce + the shard slice, which is the same arithmetic."""

    def __init__(self, prims, grads_cls, group=None):
        from .primitive import FlatGroups

        self.group = group
        self.world = torch.distributed.get_world_size(group)
        self.rank = torch.distributed.get_rank(group)
        p = prims.flat
        self.total = p.numel()
        quantum = 4 * self.world
        self.padded = -(-self.total // quantum) * quantum
        self.shard = self.padded // self.world
        self.lo = self.rank * self.shard
        pbuf = torch.zeros(self.padded, dtype=p.dtype, device=p.device)
        pbuf[: self.total].copy_(p)
        FlatGroups.__init__(prims, prims.n, prims.k, pbuf[: self.total], prims.lobes)  # re-home in place
        self.pbuf = pbuf
        self.gbuf = torch.zeros(self.padded, dtype=p.dtype, device=p.device)
        self.grads = grads_cls(prims.n, prims.k, flat=self.gbuf[: self.total], lobes=prims.lobes)
        self.gshard = torch.zeros(self.shard, dtype=p.dtype, device=p.device)
        self.exp_avg = torch.zeros(self.shard, dtype=p.dtype, device=p.device)
        self.exp_avg_sq = torch.zeros(self.shard, dtype=p.dtype, device=p.device)
        self._step_buf = torch.zeros(2, dtype=torch.int64, device=p.device)
        self.step_dev = self._step_buf[:1]
        self.prims = prims
        self.native = torch.distributed.get_backend(group) == "nccl"

    def shard_group_ends(self):
        """Global group ends shifted into the shard's coordinates (clipped to [0, S])."""
        return [min(max(e - self.lo, 0), self.shard) for e in self.prims.group_ends()]

    def reduce_scatter(self):
        if self.native:
            torch.distributed.reduce_scatter_tensor(self.gshard, self.gbuf, group=self.group)
        else:  # host-side collective (gloo): same sum, then this rank's slice
            g = self.gbuf.cpu()
            torch.distributed.all_reduce(g, group=self.group)
            self.gshard.copy_(g[self.lo: self.lo + self.shard])

    def all_gather(self):
        mine = self.pbuf[self.lo: self.lo + self.shard]
        if self.native:
            torch.distributed.all_gather_into_tensor(self.pbuf, mine, group=self.group)
        else:
            parts = [torch.empty(self.shard, dtype=self.pbuf.dtype) for _ in range(self.world)]
            torch.distributed.all_gather(parts, mine.cpu(), group=self.group)
            self.pbuf.copy_(torch.cat(parts).to(self.pbuf.device))
