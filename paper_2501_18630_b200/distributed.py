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
