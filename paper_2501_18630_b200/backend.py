"""Raster-core selection: the reference's plugin seam (backend.py:28-42).

``get_core(name)`` resolves ``None`` through ``BETASPLAT_BACKEND`` exactly like the
reference; this package provides one core, ``"cuda"`` (``"auto"`` maps to it).  Unknown
names raise ValueError; asking for the cuda core without a built library or without a
CUDA device raises RuntimeError -- there is no CPU fallback.
"""

from __future__ import annotations

import os

from . import _lib


def have_cuda_core() -> bool:
    try:
        import torch

        return os.path.exists(_lib.LIB_PATH) and torch.cuda.is_available()
    except Exception:
        return False


def available_backends():
    return ["cuda"] if have_cuda_core() else []


def get_core(name=None):
    if name is None:
        name = os.environ.get("BETASPLAT_BACKEND", "auto")
    if name in ("auto", "cuda"):
        _lib.require_cuda()
        from . import cuda_core

        return cuda_core
    raise ValueError(f"unknown backend {name!r} (expected cuda/auto)")


def active_backend():
    return "cuda"
