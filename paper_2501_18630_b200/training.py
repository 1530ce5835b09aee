"""Training step on the device: loss, Adam, and the view-batch step (configs 1, 3, 4).

``loss`` / ``adam_step`` mirror training.loss / training.adam_step
(training.py:98-131, 258-273) through libbsr kernels (K7, K8).  ``TrainStep`` is the
per-iteration hot path a user of the reference's ``train`` loop (training.py:357-366)
switches to:

    for each view of this rank:  render_tiled -> loss -> render_backward (accumulate)
    [all-reduce of the flat gradient buffer over NCCL when world_size > 1]
    fused Adam with per-group learning rates

The sort is treated as locally constant and every kernel is stream ordered; no host
synchronisation happens inside ``step(check=False)``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .camera import Camera
from .distributed import allreduce_grads
from .primitive import GradientBuffer, PrimitiveSet
from .rasterizer import (FrameState, _bg_arr, _prims_scene_c, backward_raw, forward_raw, frame_status,
                         grads_c, outputs_c)

ADAM_BETA1 = 0.9  # training.py:31
ADAM_BETA2 = 0.999  # training.py:32
ADAM_EPS = 1e-15  # training.py:33


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class LossWorkspace:
    def __init__(self, width, height, device="cuda"):
        out = ctypes.c_uint64()
        _lib.check(_lib.load().bsr_loss_scratch_bytes(width, height, ctypes.byref(out)), "loss")
        self.nbytes = int(out.value)
        self.scratch = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.values = torch.zeros(3, dtype=torch.float64, device=device)
        self.width, self.height = width, height


def loss_into(rendered, target, d_image, ws: LossWorkspace, lambda_ssim=0.2, raw=None):
    """Device-side loss: writes d_image (optionally masked by raw >= 0) and ws.values =
    [loss, l1, ssim] without a host sync."""
    h, w = rendered.shape[:2]
    rc = _lib.load().bsr_loss_l1_dssim(
        rendered.data_ptr(), target.data_ptr(), _lib.ptr(raw), w, h, float(lambda_ssim),
        ws.values.data_ptr(), d_image.data_ptr(), ws.scratch.data_ptr(), ws.nbytes, _stream())
    _lib.check(rc, "loss")


def loss(rendered, target, lambda_ssim=0.2):
    """training.loss with lambda_opacity = lambda_scale = 0: returns (value, d_image)."""
    _lib.require_cuda()
    rendered = torch.as_tensor(rendered, dtype=torch.float32, device="cuda").contiguous()
    target = torch.as_tensor(target, dtype=torch.float32, device="cuda").contiguous()
    if rendered.shape != target.shape:
        raise ValueError("rendered/target shapes differ")
    if rendered.dim() != 3 or rendered.shape[2] != 3:
        raise ValueError("images must be (H, W, 3)")
    if rendered.shape[0] < 11 or rendered.shape[1] < 11:
        raise ValueError("images must be at least 11x11")
    ws = LossWorkspace(rendered.shape[1], rendered.shape[0])
    d_image = torch.empty_like(rendered)
    loss_into(rendered, target, d_image, ws, lambda_ssim)
    vals = ws.values.cpu().numpy()
    return float(vals[0]), d_image


def ssim(a, b):
    """Mean SSIM (training.py:51-83) via the loss kernel with lambda = 1."""
    a = torch.as_tensor(a, dtype=torch.float32, device="cuda").contiguous()
    b = torch.as_tensor(b, dtype=torch.float32, device="cuda").contiguous()
    ws = LossWorkspace(a.shape[1], a.shape[0])
    d = torch.empty_like(a)
    loss_into(a, b, d, ws, 1.0)
    return float(ws.values[2].item()), -d


class AdamState:
    """First/second moments as flat buffers aligned with the PrimitiveSet (training.py:230-255)."""

    def __init__(self, prims: PrimitiveSet):
        self.exp_avg = torch.zeros_like(prims.flat)
        self.exp_avg_sq = torch.zeros_like(prims.flat)
        self.step = 0
        # device-side step counter for graph-captured steps (bsr_adam_step_device)
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=prims.flat.device)


def sb_group_lrs(lr_means=1.6e-4):
    """The reference's default per-group learning rates (TrainConfig.group_lrs,
    training.py:217-227) for a Spherical-Beta set."""
    return {"positions": lr_means, "opacity_raw": 5e-2, "rotations": 1e-3, "log_scales": 5e-3,
            "shapes": 1e-3, "base_colors": 2.5e-3, "lobe_axes": 2.5e-3, "lobe_colors": 2.5e-3}


def group_lrs(lr_means=1.6e-4, lr_other=5e-3, lr_shapes=0.0):
    """Config-3 learning rates (BASELINE.json configs[3]): 1.6e-4 for means, 5e-3 for the
    other optimised attributes (quats, scales, opacities, SH).  The configs render the
    Gaussian-like kernel (b = 0, beta = 4) and do not list the Beta shape among the
    optimised attributes, so ``shapes`` is frozen by default (lr 0); pass lr_shapes to
    train it like the reference's full DBS optimiser (training.py:217-227)."""
    return {"positions": lr_means, "rotations": lr_other, "log_scales": lr_other, "opacity_raw": lr_other,
            "shapes": lr_shapes, "sh": lr_other}


def adam_step(prims: PrimitiveSet, grads: GradientBuffer, state: AdamState, lrs: dict,
              device_step: bool = False):
    """training.py:258-273 as one fused kernel over the flat buffers.

    ``device_step`` keeps the step count on the device (graph-capturable); the host-side
    ``state.step`` then only counts calls made outside captured graphs."""
    groups = prims.groups
    ends = (ctypes.c_int64 * len(groups))(*prims.group_ends())
    lr = (ctypes.c_float * len(groups))(*[float(lrs[g]) for g in groups])
    lib = _lib.load()
    if device_step:
        rc = lib.bsr_adam_step_device(prims.flat.data_ptr(), grads.flat.data_ptr(), state.exp_avg.data_ptr(),
                                      state.exp_avg_sq.data_ptr(), prims.flat.numel(), len(groups), ends, lr,
                                      state.step_dev.data_ptr(), ADAM_BETA1, ADAM_BETA2, ADAM_EPS, _stream())
    else:
        state.step += 1
        state.step_dev.fill_(state.step)
        rc = lib.bsr_adam_step(prims.flat.data_ptr(), grads.flat.data_ptr(), state.exp_avg.data_ptr(),
                               state.exp_avg_sq.data_ptr(), prims.flat.numel(), len(groups), ends, lr, state.step,
                               ADAM_BETA1, ADAM_BETA2, ADAM_EPS, _stream())
    _lib.check(rc, "adam")
    return prims


class TrainStep:
    """One training iteration over this rank's views (fwd + L1/D-SSIM + bwd [+ all-reduce] + Adam)."""

    def __init__(self, prims: PrimitiveSet, cameras: list, targets: list, background, lrs=None,
                 lambda_ssim=0.2, process_group=None):
        self.prims = prims
        self.cameras = list(cameras)
        self.targets = list(targets)
        self.background = background
        self.lrs = lrs or (group_lrs() if prims.color_model == "sh" else sb_group_lrs())
        self.lambda_ssim = lambda_ssim
        self.pg = process_group
        self.grads = GradientBuffer.zeros_for(prims)
        self.adam = AdamState(prims)
        self.scene = _prims_scene_c(prims)
        self.gc = grads_c(self.grads)
        dev = prims.flat.device
        self.frames: dict = {}
        self.bufs = {}
        self.loss_ws = {}
        for cam in self.cameras:
            key = (cam.width, cam.height)
            if key not in self.bufs:
                h, w = cam.height, cam.width
                self.bufs[key] = dict(color=torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                                      d_image=torch.empty((h, w, 3), dtype=torch.float32, device=dev))
                self.loss_ws[key] = LossWorkspace(w, h, dev)
        self.loss_values = torch.zeros((len(self.cameras), 3), dtype=torch.float64, device=dev)
        self.profile = None  # optional rasterizer.StageProfiler-like object with .fwd/.bwd

    def _frame(self, cam):
        return self.frames.get((cam.width, cam.height))

    def step(self, check=False, adam=True):
        prof = self.profile
        self.grads.flat.zero_()
        for i, (cam, target) in enumerate(zip(self.cameras, self.targets)):
            key = (cam.width, cam.height)
            b = self.bufs[key]
            frame = forward_raw(self.scene, cam, self.background, outputs_c(color=b["color"]),
                                frame=self._frame(cam), check=check,
                                profile=None if prof is None else prof.fwd(i))
            self.frames[key] = frame
            ws = self.loss_ws[key]
            if prof is not None:
                prof.mark_loss(i)
            loss_into(b["color"], target, b["d_image"], ws, self.lambda_ssim)
            if prof is not None:
                prof.mark_loss(i, end=True)
            self.loss_values[i].copy_(ws.values)
            backward_raw(self.scene, cam, self.background, frame, b["d_image"], None, self.gc, None,
                         profile=None if prof is None else prof.bwd(i))
        if self.pg is not None:  # the one exchange step of view-batch DP (distributed.py)
            allreduce_grads(self.grads.flat, group=self.pg)
        if adam:
            if prof is not None:
                prof.mark_adam()
            adam_step(self.prims, self.grads, self.adam, self.lrs, device_step=True)
            if prof is not None:
                prof.mark_adam(end=True)
        return self.loss_values

    def capture(self, adam=True, warmup=2):
        """Capture one whole step (every view's fwd + loss + bwd [+ all-reduce] + Adam) in a
        CUDA graph: ~30 kernel launches become one graph launch.  Frames must already be
        sized (run step(check=True) once first); capacity is re-checked by check_frames()."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self.step(check=False, adam=adam)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.step(check=False, adam=adam)
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.loss_values

    def check_frames(self):
        """Host-side check of every frame's device status (capacity / errors)."""
        for f in self.frames.values():
            frame_status(f)


def render_targets(target_prims: PrimitiveSet, cameras, background):
    """Per-view target images rendered once on the device (configs 1, 3)."""
    from .rasterizer import render_tiled

    return [render_tiled(target_prims, cam, background).color.contiguous() for cam in cameras]


__all__ = ["loss", "ssim", "adam_step", "AdamState", "TrainStep", "render_targets", "group_lrs",
           "LossWorkspace", "loss_into", "FrameState", "Camera", "np", "_bg_arr"]
