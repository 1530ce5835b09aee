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
from dataclasses import dataclass, field, fields

import numpy as np
import torch

from . import _lib
from .camera import Camera
from .distributed import allreduce_grads
from .primitive import GradientBuffer, PrimitiveSet
from .rasterizer import (FrameState, _bg_arr, _prims_scene_c, backward_raw, color_grad_views, det_workspace, forward_raw,
                         frame_status, grads_c, outputs_c)

ADAM_BETA1 = 0.9  # training.py:31
ADAM_BETA2 = 0.999  # training.py:32
ADAM_EPS = 1e-15  # training.py:33


def _stream():
    return _lib.stream_ptr()


class LossWorkspace:
    def __init__(self, width, height, device="cuda"):
        out = ctypes.c_uint64()
        _lib.check(_lib.load().bsr_loss_scratch_bytes(width, height, ctypes.byref(out)), "loss")
        self.nbytes = int(out.value)
        self.scratch = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.values = torch.zeros(3, dtype=torch.float64, device=device)
        self.width, self.height = width, height


def loss_into(rendered, target, d_image, ws: LossWorkspace, lambda_ssim=0.2, raw=None, values=None):
    """Device-side loss: writes d_image (optionally masked by raw >= 0) and [loss, l1, ssim]
    into ``values`` (3 float64 on the device; default ws.values) without a host sync."""
    h, w = rendered.shape[:2]
    out = ws.values if values is None else values
    rc = _lib.load().bsr_loss_l1_dssim(
        rendered.data_ptr(), target.data_ptr(), _lib.ptr(raw), w, h, float(lambda_ssim),
        out.data_ptr(), d_image.data_ptr(), ws.scratch.data_ptr(), ws.nbytes, _stream())
    _lib.check(rc, "loss")


def regularizers_into(prims: PrimitiveSet, grads: GradientBuffer, lambda_opacity: float, lambda_scale: float,
                      loss_out=None):
    """training.loss direct terms (training.py:112-124) on the device: grads.opacity_raw +=
    lo * o (1 - o), grads.log_scales += ls * s; loss_out[0] += lo * sum(o) + ls * sum(s)."""
    lc = prims.layout_c()
    rc = _lib.load().bsr_regularizers(prims.flat.data_ptr(), ctypes.byref(lc), float(lambda_opacity),
                                      float(lambda_scale), grads.flat.data_ptr(), _lib.ptr(loss_out), _stream())
    _lib.check(rc, "regularizers")


def loss(rendered, target, prims=None, cfg=None, return_parts=False, lambda_ssim=None):
    """training.loss (training.py:98-131).

    ``loss(rendered, target)`` -> (value, d_image) with lambda_ssim = 0.2 and no
    regularisers (the BASELINE configs).  With ``prims`` (and optionally a TrainConfig
    ``cfg``) it returns the reference's ``(value, d_image, direct[, parts])``: ``direct``
    holds the opacity / log-scale regulariser gradients as device tensors."""
    lam = (cfg.lambda_ssim if cfg is not None else 0.2) if lambda_ssim is None else lambda_ssim
    if prims is None:
        return _image_loss(rendered, target, lam)
    _lib.require_cuda()
    lo = cfg.lambda_opacity if cfg is not None else TrainConfig.lambda_opacity
    ls = cfg.lambda_scale if cfg is not None else TrainConfig.lambda_scale
    rendered = torch.as_tensor(rendered, dtype=torch.float32, device="cuda").contiguous()
    target = torch.as_tensor(target, dtype=torch.float32, device="cuda").contiguous()
    _check_images(rendered, target)
    ws = LossWorkspace(rendered.shape[1], rendered.shape[0])
    d_image = torch.empty_like(rendered)
    loss_into(rendered, target, d_image, ws, lam)
    g = GradientBuffer.zeros_for(prims)
    regularizers_into(prims, g, lo, ls, ws.values)
    vals = ws.values.cpu().numpy()
    direct = {"opacity_raw": g.opacity_raw, "log_scales": g.log_scales}
    if return_parts:
        return float(vals[0]), d_image, direct, {"l1": float(vals[1]), "ssim_term": 1.0 - float(vals[2])}
    return float(vals[0]), d_image, direct


def _check_images(rendered, target):
    if rendered.shape != target.shape:
        raise ValueError("rendered/target shapes differ")
    if rendered.dim() != 3 or rendered.shape[2] != 3:
        raise ValueError("images must be (H, W, 3)")
    if rendered.shape[0] < 11 or rendered.shape[1] < 11:
        raise ValueError("images must be at least 11x11")


def _image_loss(rendered, target, lambda_ssim=0.2):
    """training.loss with lambda_opacity = lambda_scale = 0: returns (value, d_image)."""
    _lib.require_cuda()
    rendered = torch.as_tensor(rendered, dtype=torch.float32, device="cuda").contiguous()
    target = torch.as_tensor(target, dtype=torch.float32, device="cuda").contiguous()
    _check_images(rendered, target)
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
        # device-side step counter for graph-captured steps: [0] the step, [1] the fused
        # kernel's block ticket (bsr_adam_step_fused)
        self._step_buf = torch.zeros(2, dtype=torch.int64, device=prims.flat.device)
        self.step_dev = self._step_buf[:1]
        self._prims = prims

    @classmethod
    def zeros_for(cls, prims: PrimitiveSet) -> "AdamState":
        return cls(prims)

    def zero_rows(self, indices):
        """Zero both moments of the given primitives in every group (training.py:243-246)."""
        idx = torch.as_tensor(indices, dtype=torch.long, device=self.exp_avg.device)
        p = self._prims
        for buf in (self.exp_avg, self.exp_avg_sq):
            view = PrimitiveSet.from_flat(p.n, p.k, buf, p.lobes)
            for g in view.groups:
                getattr(view, g)[idx] = 0.0


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
              device_step: bool = False, schedule=None, zero_grads: bool = False):
    """training.py:258-273 as one fused kernel over the flat buffers.

    ``device_step`` keeps the step count on the device (graph-capturable); the host-side
    ``state.step`` then only counts calls made outside captured graphs.  ``zero_grads``
    (device_step only) clears the gradients as the kernel consumes them, so the next step
    needs no separate memset."""
    groups = prims.groups
    ends = (ctypes.c_int64 * len(groups))(*prims.group_ends())
    lr = (ctypes.c_float * len(groups))(*[float(lrs[g]) for g in groups])
    lib = _lib.load()
    if device_step:  # one kernel: bias corrections from, and bump of, the device counter
        rc = lib.bsr_adam_step_fused(prims.flat.data_ptr(), grads.flat.data_ptr(), state.exp_avg.data_ptr(),
                                     state.exp_avg_sq.data_ptr(), prims.flat.numel(), len(groups), ends, lr,
                                     state._step_buf.data_ptr(),
                                     None if schedule is None else ctypes.byref(schedule),
                                     groups.index("positions") if schedule is not None else -1,
                                     ADAM_BETA1, ADAM_BETA2, ADAM_EPS, int(bool(zero_grads)), _stream())
    elif schedule is not None:  # positions follow the lr schedule at the device step
        rc = lib.bsr_adam_step_scheduled(prims.flat.data_ptr(), grads.flat.data_ptr(), state.exp_avg.data_ptr(),
                                         state.exp_avg_sq.data_ptr(), prims.flat.numel(), len(groups), ends, lr,
                                         state.step_dev.data_ptr(), ctypes.byref(schedule),
                                         groups.index("positions"), ADAM_BETA1, ADAM_BETA2, ADAM_EPS, _stream())
    else:
        state.step += 1
        state.step_dev.fill_(state.step)
        rc = lib.bsr_adam_step(prims.flat.data_ptr(), grads.flat.data_ptr(), state.exp_avg.data_ptr(),
                               state.exp_avg_sq.data_ptr(), prims.flat.numel(), len(groups), ends, lr, state.step,
                               ADAM_BETA1, ADAM_BETA2, ADAM_EPS, _stream())
    _lib.check(rc, "adam")
    return prims


# ----------------------------------------------------------------------------- schedules
def _sched_c(lr_init, lr_final, max_steps, delay_steps=0, delay_mult=0.01, scale=1.0):
    c = _lib.LrScheduleC()
    c.lr_init, c.lr_final, c.max_steps = float(lr_init), float(lr_final), int(max_steps)
    c.delay_steps, c.delay_mult, c.scale = int(delay_steps), float(delay_mult), float(scale)
    return c


def exponential_lr(step, lr_init, lr_final, max_steps, delay_steps=0, delay_mult=0.01):
    """Log-linear interpolation from init to final over ``max_steps`` (training.py:134-145),
    evaluated by the same code the device uses inside Adam / inject_noise."""
    c = _sched_c(lr_init, lr_final, max_steps, delay_steps, delay_mult)
    return float(_lib.load().bsr_scheduled_lr(ctypes.byref(c), int(step)))


@dataclass
class TrainConfig:
    """Hyperparameters of the reference's optimiser (training.py:148-204); field names
    double as config-file keys.  Only the fields the device training step uses are
    consumed here; the rest are carried for drop-in compatibility."""

    lambda_ssim: float = 0.2
    lambda_opacity: float = 0.01
    lambda_scale: float = 0.01
    noise_lr: float = 5e4
    lr_position_init: float = 1.6e-4
    lr_position_final: float = 1.6e-6
    lr_position_delay_steps: int = 0
    lr_position_delay_mult: float = 0.01
    lr_position_max_steps: int = 30_000
    lr_base_color: float = 2.5e-3
    lr_lobes: float = 2.5e-3
    lr_opacity: float = 5e-2
    lr_shape: float = 1e-3
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    lr_sh: float = 2.5e-3
    densify_interval: int = 100
    densify_start: int = 500
    densify_end: int = 25_000
    dead_threshold: float = 0.005
    growth_rate: float = 0.05
    max_primitives: int = 1_000_000
    total_steps: int = 30_000
    patience: int = 10_000
    mode: str = "30k"
    sb_lobes: int = 2
    init_opacity: float = 0.1
    init_count: int = 2000
    init_mode: str = "auto"
    scene_scale: float = 0.0
    background: str = "white"
    holdout: int = 8
    eval_interval: int = 250
    max_steps_cap: int = 300_000

    def __post_init__(self):
        for f in fields(self):
            if f.name.startswith("lr_") and f.name not in ("lr_position_delay_steps", "lr_position_delay_mult",
                                                            "lr_position_max_steps"):
                if getattr(self, f.name) <= 0:
                    raise ValueError(f"{f.name} must be positive")
        if self.densify_start >= self.densify_end:
            raise ValueError("densify_start must be below densify_end")
        if self.mode not in ("30k", "full"):
            raise ValueError("mode must be '30k' or 'full'")

    def background_rgb(self):
        if self.background == "white":
            return np.ones(3)
        if self.background == "black":
            return np.zeros(3)
        return np.array([float(v) for v in self.background.split(",")], dtype=np.float64)

    def position_schedule(self, scene_scale=1.0):
        return _sched_c(self.lr_position_init, self.lr_position_final, self.lr_position_max_steps,
                        self.lr_position_delay_steps, self.lr_position_delay_mult, scene_scale)

    def position_lr(self, step, scene_scale=1.0):
        return scene_scale * exponential_lr(step, self.lr_position_init, self.lr_position_final,
                                            self.lr_position_max_steps, self.lr_position_delay_steps,
                                            self.lr_position_delay_mult)

    def group_lrs(self, step, scene_scale=1.0):
        return {"positions": self.position_lr(step, scene_scale), "opacity_raw": self.lr_opacity,
                "rotations": self.lr_rotation, "log_scales": self.lr_scale, "shapes": self.lr_shape,
                "base_colors": self.lr_base_color, "lobe_axes": self.lr_lobes, "lobe_colors": self.lr_lobes,
                "sh": self.lr_sh}


def inject_noise(prims: PrimitiveSet, cfg: TrainConfig, position_lr, rng, step_counter=None, schedule=None):
    """Covariance-shaped, opacity-gated position noise (training.py:276-292), in place.

    ``rng``: a numpy Generator (eta = rng.standard_normal((n, 3)), the reference's draw) or
    an ``mcmc.DeviceRNG`` (Philox on the device, keyed by the device step counter when one
    is given, so a captured graph draws fresh noise every replay)."""
    from .mcmc import DeviceRNG

    n = len(prims)
    if n == 0:
        return prims.positions
    lc = prims.layout_c()
    eta = None
    seed = offset = 0
    if isinstance(rng, DeviceRNG):
        seed = rng.seed
        # step-keyed draws live in their own reserved counter range (never the MCMC draws')
        offset = rng.advance(1 << 32) if step_counter is None else rng.domain("noise")
    else:
        eta = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((n, 3)), dtype=np.float32)).to(
            prims.flat.device)
    status = torch.zeros(1, dtype=torch.int32, device=prims.flat.device)
    rc = _lib.load().bsr_inject_noise(prims.flat.data_ptr(), ctypes.byref(lc), float(cfg.noise_lr),
                                      float(position_lr if position_lr is not None else 0.0),
                                      None if schedule is None else ctypes.byref(schedule),
                                      _lib.ptr(step_counter), _lib.ptr(eta), seed, offset, status.data_ptr(),
                                      _stream())
    _lib.check(rc, "inject_noise")
    if step_counter is None and int(status.item()) != 0:
        _lib.check(int(status.item()), "inject_noise")
    return prims.positions


class TrainStep:
    """One training iteration over this rank's views (fwd + L1/D-SSIM + bwd [+ all-reduce] + Adam)."""

    def __init__(self, prims: PrimitiveSet, cameras: list, targets: list, background, lrs=None,
                 lambda_ssim=0.2, process_group=None, cfg: TrainConfig | None = None, scene_scale=1.0,
                 noise_rng=None, defer_color=True, deterministic=False, shard_optimizer=True,
                 precompute_colors=True):
        """``cfg`` switches on the reference's full optimiser step (training.py:357-366):
        opacity / scale regularisers, the exponential position-lr schedule and the
        covariance-shaped position noise, all evaluated on the device from the device step
        counter (graph-capturable).  Without it the step is the BASELINE configs' (L1 +
        D-SSIM, constant group learning rates, no noise).  ``deterministic`` runs every
        view's backward in the fixed-point mode (bsr_backward_deterministic): the whole step,
        Adam included, is bitwise reproducible on one GPU.  With a ``process_group`` the
        exchange is reduce-scatter -> Adam on this rank's shard -> all-gather
        (distributed.ShardedOptimizer) unless ``shard_optimizer`` is False (all-reduce +
        replicated Adam)."""
        self.prims = prims
        self.cfg = cfg
        self.scene_scale = float(scene_scale)
        if cfg is not None:
            from .mcmc import DeviceRNG

            lambda_ssim = cfg.lambda_ssim
            lrs = lrs or cfg.group_lrs(0, scene_scale)
            self.noise_rng = noise_rng or DeviceRNG(0)
            self.noise_offset = self.noise_rng.advance(1 << 40)
            self.schedule = cfg.position_schedule(scene_scale)
            self.rank0 = process_group is None or torch.distributed.get_rank(process_group) == 0
        self.cameras = list(cameras)
        self.targets = list(targets)
        self.background = background
        self.lrs = lrs or (group_lrs() if prims.color_model == "sh" else sb_group_lrs())
        self.lambda_ssim = lambda_ssim
        self.pg = process_group
        self.sharded = None
        if process_group is not None and shard_optimizer:
            from .distributed import ShardedOptimizer

            self.sharded = ShardedOptimizer(prims, GradientBuffer, process_group)
            self.grads = self.sharded.grads
            self.adam = self.sharded  # exp_avg / exp_avg_sq / step_dev of this rank's shard
        else:
            self.grads = GradientBuffer.zeros_for(prims)
            self.adam = AdamState(prims)
        self.scene = _prims_scene_c(prims)
        self.gc = grads_c(self.grads)
        # one view without a deferred colour chain: its backward WRITES the gradient buffer
        # (bsr_grads::overwrite), so the step needs no memset of it
        self.gc_write = grads_c(self.grads, overwrite=True)
        self.write_first = len(self.cameras) == 1 and self.sharded is None
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
        # several views of an SH set: each view's backward defers its colour chain into
        # drgb[v] and one kernel applies them all after the last view (the 3K coefficient
        # gradients are read and written once per step instead of once per view)
        self.drgb = None
        if len(self.cameras) > 1 and prims.color_model == "sh" and defer_color:
            self.drgb = torch.empty((len(self.cameras), prims.n, 4), dtype=torch.float32, device=dev)
        self.det_ws = det_workspace(prims.n, dev) if deterministic else None
        # several views: the colours of every view are evaluated in one pass over the
        # appearance parameters (bsr_view_colors) at the start of the step, and each view's
        # forward reads its (N, 4) slice instead of the SH coefficients (bsr_scene.view_rgb)
        self.vrgb = None
        if len(self.cameras) > 1 and precompute_colors:
            self.vrgb = torch.empty((len(self.cameras), prims.n, 4), dtype=torch.float32, device=dev)
            self.view_scenes = []
            for v in range(len(self.cameras)):
                sv = _lib.SceneC.from_buffer_copy(self.scene)
                sv.view_rgb = self.vrgb[v].data_ptr()
                self.view_scenes.append(sv)
            self.centers = np.ascontiguousarray(np.stack([np.asarray(c.center, np.float64) for c in self.cameras]))
        self.profile = None  # optional rasterizer.StageProfiler-like object with .fwd/.bwd
        self._grads_clear = False  # the last step's Adam zeroed self.grads

    def _frame(self, cam):
        return self.frames.get((cam.width, cam.height))

    def step(self, check=False, adam=True):
        prof = self.profile
        write = self.write_first and self.drgb is None
        if not self._grads_clear and not write:
            self.grads.flat.zero_()
        self._grads_clear = False
        if self.vrgb is not None:
            _lib.check(_lib.load().bsr_view_colors(ctypes.byref(self.scene), self.centers.ctypes.data_as(ctypes.c_void_p),
                                                   len(self.cameras), self.vrgb.data_ptr(), _stream()), "view_colors")
        for i, (cam, target) in enumerate(zip(self.cameras, self.targets)):
            key = (cam.width, cam.height)
            b = self.bufs[key]
            frame = forward_raw(self.scene if self.vrgb is None else self.view_scenes[i], cam, self.background,
                                outputs_c(color=b["color"]),
                                frame=self._frame(cam), check=check,
                                profile=None if prof is None else prof.fwd(i))
            self.frames[key] = frame
            ws = self.loss_ws[key]
            if prof is not None:
                prof.mark_loss(i)
            loss_into(b["color"], target, b["d_image"], ws, self.lambda_ssim, values=self.loss_values[i])
            if prof is not None:
                prof.mark_loss(i, end=True)
            backward_raw(self.scene, cam, self.background, frame, b["d_image"], None,
                         self.gc_write if (write and i == 0) else self.gc, None,
                         profile=None if prof is None else prof.bwd(i),
                         drgb=None if self.drgb is None else self.drgb[i], det_ws=self.det_ws)
        if self.drgb is not None:
            if prof is not None and hasattr(prof, "mark_color"):
                prof.mark_color()
            color_grad_views(self.scene, self.drgb, self.cameras, self.gc)
            if prof is not None and hasattr(prof, "mark_color"):
                prof.mark_color(end=True)
        cfg = self.cfg
        if cfg is not None and self.rank0:  # direct regulariser terms, once per iteration
            regularizers_into(self.prims, self.grads, cfg.lambda_opacity, cfg.lambda_scale, self.loss_values[0])
        if self.sharded is not None:  # reduce-scatter -> sharded Adam -> all-gather (distributed.py)
            if prof is not None:
                prof.mark_adam()
            sh = self.sharded
            sh.reduce_scatter()
            if adam:
                _sharded_adam(sh, self.lrs, None if cfg is None else self.schedule)
                sh.all_gather()
            sh.gbuf.zero_()  # the next step accumulates from zero
            self._grads_clear = True
            if adam and cfg is not None:
                lc = self.prims.layout_c()
                rc = _lib.load().bsr_inject_noise(self.prims.flat.data_ptr(), ctypes.byref(lc), float(cfg.noise_lr),
                                                  0.0, ctypes.byref(self.schedule), sh.step_dev.data_ptr(),
                                                  None, self.noise_rng.seed, self.noise_offset, None, _stream())
                _lib.check(rc, "inject_noise")
            if prof is not None:
                prof.mark_adam(end=True)
            return self.loss_values
        if self.pg is not None:  # the one exchange step of view-batch DP (distributed.py)
            allreduce_grads(self.grads.flat, group=self.pg)
        if adam:
            if prof is not None:
                prof.mark_adam()
            # Adam clears the gradients it consumes: the next step skips its memset
            adam_step(self.prims, self.grads, self.adam, self.lrs, device_step=True,
                      schedule=None if cfg is None else self.schedule, zero_grads=True)
            self._grads_clear = True
            if cfg is not None:
                # position noise at this step's scheduled lr (Adam bumped the device step)
                lc = self.prims.layout_c()
                rc = _lib.load().bsr_inject_noise(self.prims.flat.data_ptr(), ctypes.byref(lc), float(cfg.noise_lr),
                                                  0.0, ctypes.byref(self.schedule), self.adam.step_dev.data_ptr(),
                                                  None, self.noise_rng.seed, self.noise_offset, None, _stream())
                _lib.check(rc, "inject_noise")
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
        mode = "thread_local" if self.pg is not None else "global"  # see bench.capture_mode
        with torch.cuda.graph(self.graph, capture_error_mode=mode):
            self.step(check=False, adam=adam)
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.loss_values

    def check_frames(self):
        """Host-side check of every frame's device status (capacity / errors)."""
        for f in self.frames.values():
            frame_status(f)


def _sharded_adam(sh, lrs: dict, schedule=None):
    """The fused Adam kernel on this rank's shard (distributed.ShardedOptimizer): shard
    pointers, the global group ends shifted into shard coordinates, the device step counter
    bumped by the kernel (graph-capturable)."""
    groups = sh.prims.groups
    ends = (ctypes.c_int64 * len(groups))(*sh.shard_group_ends())
    lr = (ctypes.c_float * len(groups))(*[float(lrs[g]) for g in groups])
    p = sh.pbuf[sh.lo: sh.lo + sh.shard]
    rc = _lib.load().bsr_adam_step_fused(p.data_ptr(), sh.gshard.data_ptr(), sh.exp_avg.data_ptr(),
                                         sh.exp_avg_sq.data_ptr(), sh.shard, len(groups), ends, lr,
                                         sh._step_buf.data_ptr(),
                                         None if schedule is None else ctypes.byref(schedule),
                                         groups.index("positions") if schedule is not None else -1,
                                         ADAM_BETA1, ADAM_BETA2, ADAM_EPS, 0, _stream())
    _lib.check(rc, "adam (shard)")


def render_targets(target_prims: PrimitiveSet, cameras, background):
    """Per-view target images rendered once on the device (configs 1, 3)."""
    from .rasterizer import render_tiled

    return [render_tiled(target_prims, cam, background).color.contiguous() for cam in cameras]


# ----------------------------------------------------------------------------- train loop
@dataclass
class TrainResult:
    primitives: object
    metrics: list = field(default_factory=list)
    best_psnr: float = -np.inf
    best_step: int = 0
    steps_run: int = 0
    diverged: bool = False
    abort_reason: str = ""


def scene_scale_from_cameras(cameras):
    """training.py:307-311."""
    centers = np.stack([c.center for c in cameras])
    return max(float(np.max(np.linalg.norm(centers - centers.mean(axis=0), axis=1))), 1e-6)


def psnr(a, b):
    """``10 log10(1 / MSE)`` (training.py:86-95), reduced on the device."""
    a = torch.as_tensor(a, device="cuda", dtype=torch.float32)
    b = torch.as_tensor(b, device="cuda", dtype=torch.float32)
    if a.shape != b.shape:
        raise ValueError(f"image shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    mse = float(torch.mean((a.double() - b.double()) ** 2))
    return np.inf if mse == 0.0 else 10.0 * np.log10(1.0 / mse)


def evaluate_psnr(prims, dataset, view_ids, background):
    from .rasterizer import render_tiled

    vals = [psnr(render_tiled(prims, dataset.cameras[v], background).color, _device_image(dataset.images[v]))
            for v in view_ids]
    return float(np.mean(vals)) if vals else float("nan")


def _device_image(img):
    return torch.as_tensor(np.asarray(img) if not isinstance(img, torch.Tensor) else img, dtype=torch.float32,
                           device="cuda").contiguous()


class _Trainer:
    """Device buffers of one primitive count (rebuilt after mcmc.grow)."""

    def __init__(self, prims, cfg, scale, background):
        self.prims, self.cfg, self.background = prims, cfg, background
        self.grads = GradientBuffer.zeros_for(prims)
        self.scene = _prims_scene_c(prims)
        self.gc = grads_c(self.grads)
        self.frames, self.bufs = {}, {}
        self.schedule = cfg.position_schedule(scale)
        self.values = torch.zeros(3, dtype=torch.float64, device=prims.flat.device)

    def step(self, cam, target, adam: AdamState, lrs, noise):
        key = (cam.width, cam.height)
        if key not in self.bufs:
            h, w = cam.height, cam.width
            dev = self.prims.flat.device
            self.bufs[key] = (torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                              torch.empty((h, w, 3), dtype=torch.float32, device=dev), LossWorkspace(w, h, dev))
        color, d_img, ws = self.bufs[key]
        self.frames[key] = frame = forward_raw(self.scene, cam, self.background, outputs_c(color=color),
                                               frame=self.frames.get(key), check=True)
        loss_into(color, target, d_img, ws, self.cfg.lambda_ssim)
        self.grads.flat.zero_()
        regularizers_into(self.prims, self.grads, self.cfg.lambda_opacity, self.cfg.lambda_scale, ws.values)
        backward_raw(self.scene, cam, self.background, frame, d_img, None, self.gc, None)
        adam_step(self.prims, self.grads, adam, lrs, device_step=True, schedule=self.schedule)
        adam.step += 1
        noise(self)
        return ws.values


def _densify(prims, state, cfg, rng):
    """training.py:420-428 on the device."""
    from . import mcmc

    dead = mcmc.find_dead(prims, cfg.dead_threshold)
    if dead.numel():
        plan = mcmc.plan_relocation(prims, dead, rng, threshold=cfg.dead_threshold)
        mcmc.apply_relocation(prims, plan, state, floor=cfg.dead_threshold)
    return mcmc.grow(prims, cfg.max_primitives, rng, state, rate=cfg.growth_rate,
                     dead_threshold=cfg.dead_threshold)


def train(dataset, cfg: TrainConfig, rng, initial=None, progress=None, on_eval=None, device_rng=None):
    """The reference's training loop (training.py:314-406) with every per-step kernel on the
    device: render -> loss (+ regularisers) -> backward -> Adam (scheduled position lr)
    -> position noise, MCMC densification every ``densify_interval`` steps.

    ``dataset`` provides ``cameras``, ``images`` and ``train_indices()`` (sceneio.Dataset);
    ``initial`` is the starting PrimitiveSet (scene initialisation from SfM points is host
    I/O, outside the hot path).  ``rng`` (numpy Generator) drives the view order; the noise
    and MCMC draws use ``device_rng`` (mcmc.DeviceRNG) when given, else ``rng`` itself,
    draw for draw like the reference."""
    from . import mcmc

    if len(dataset.cameras) < 2:
        raise ValueError("training needs at least 2 views")
    train_ids = list(dataset.train_indices())
    if not train_ids:
        raise ValueError("dataset has no training views")
    if initial is None:
        raise ValueError("train() needs initial primitives (scene initialisation is host I/O)")
    _lib.require_cuda()
    val_ids = train_ids
    prims = initial.copy()
    scale = cfg.scene_scale or scene_scale_from_cameras(dataset.cameras)
    background = cfg.background_rgb()
    state = AdamState(prims)
    result = TrainResult(primitives=prims)
    targets = {v: _device_image(dataset.images[v]) for v in train_ids}
    drng = device_rng if device_rng is not None else rng
    tr = _Trainer(prims, cfg, scale, background)

    def noise(t):
        if isinstance(drng, mcmc.DeviceRNG):
            inject_noise(t.prims, cfg, None, drng, step_counter=state.step_dev, schedule=t.schedule)
        else:
            inject_noise(t.prims, cfg, cfg.position_lr(state.step, scale), drng)

    order, step = [], 0
    while True:
        if cfg.mode == "30k":
            if step >= cfg.total_steps:
                break
        else:
            plateaued = step - result.best_step >= cfg.patience
            if (step >= cfg.total_steps and plateaued) or step >= cfg.max_steps_cap:
                break
        step += 1
        if not order:
            order = [int(i) for i in rng.permutation(train_ids)]
        view = order.pop()
        vals = tr.step(dataset.cameras[view], targets[view], state, cfg.group_lrs(step, scale), noise)
        if cfg.densify_start <= step <= cfg.densify_end and step % cfg.densify_interval == 0:
            try:
                grown = _densify(prims, state, cfg, drng)
            except mcmc.AllDeadError as exc:
                result.diverged, result.abort_reason = True, str(exc)
                break
            if grown is not prims:
                prims = grown
                state._prims = prims
                tr = _Trainer(prims, cfg, scale, background)
            result.primitives = prims
        v = vals.cpu().numpy()
        row = {"step": step, "loss": float(v[0]), "l1": float(v[1]), "ssim_term": 1.0 - float(v[2]),
               "mean_opacity": float(prims.opacities.mean()), "count": len(prims), "psnr": ""}
        if step % cfg.eval_interval == 0 or step == 1:
            val_psnr = evaluate_psnr(prims, dataset, val_ids, background)
            row["psnr"] = val_psnr
            if val_psnr > result.best_psnr:
                result.best_psnr, result.best_step = val_psnr, step
            if on_eval is not None:
                on_eval(step, prims)
        result.metrics.append(row)
        if progress is not None:
            progress(row)
    result.steps_run = step
    result.primitives = prims
    return result


__all__ = ["loss", "ssim", "adam_step", "AdamState", "TrainStep", "render_targets", "group_lrs",
           "LossWorkspace", "loss_into", "FrameState", "Camera", "np", "_bg_arr", "TrainConfig", "TrainResult",
           "exponential_lr", "inject_noise", "regularizers_into", "train", "evaluate_psnr", "psnr",
           "scene_scale_from_cameras"]
