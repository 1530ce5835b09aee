"""ctypes binding of libbsr.so (the C-ABI declared in include/bsr.h).

The shared library is built in-tree (``make -C paper_2501_18630_b200/csrc`` or
``__graft_entry__.build()``).  There is no CPU fallback: if the library or a CUDA device
is missing, every compute entry point raises.  Status codes map to the reference's
exception types (ValueError for bad arguments, DegenerateQuaternionError, RuntimeError).
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbsr.so")

BSR_OK = 0
BSR_ERR_BAD_ARG = 1
BSR_ERR_CAPACITY = 2
BSR_ERR_CUDA = 3
BSR_ERR_DEGENERATE_QUAT = 4
BSR_ERR_FRAME_TOO_SMALL = 5

c_void_p, c_int32, c_int64, c_uint64, c_double, c_float = (
    ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_float)


class DegenerateQuaternionError(ValueError):
    """primitive.py:44-45 of the reference."""


class CapacityError(RuntimeError):
    def __init__(self, needed):
        super().__init__(f"tile-entry capacity exceeded (need {needed})")
        self.needed = needed


class CameraC(ctypes.Structure):
    _fields_ = [("world_to_camera", c_double * 16), ("fx", c_double), ("fy", c_double),
                ("cx", c_double), ("cy", c_double), ("width", c_int32), ("height", c_int32)]


BSR_COLOR_SH = 0
BSR_COLOR_SB = 1


class SceneC(ctypes.Structure):
    _fields_ = [("positions", c_void_p), ("rotations", c_void_p), ("log_scales", c_void_p),
                ("opacity_raw", c_void_p), ("shapes", c_void_p), ("sh", c_void_p), ("n", c_int64),
                ("sh_coeffs", c_int32), ("color_model", c_int32), ("base_colors", c_void_p),
                ("lobe_axes", c_void_p), ("lobe_colors", c_void_p), ("lobes", c_int32),
                ("reserved", c_int32), ("view_rgb", c_void_p)]


class GradsC(ctypes.Structure):
    _fields_ = [("positions", c_void_p), ("rotations", c_void_p), ("log_scales", c_void_p),
                ("opacity_raw", c_void_p), ("shapes", c_void_p), ("sh", c_void_p),
                ("base_colors", c_void_p), ("lobe_axes", c_void_p), ("lobe_colors", c_void_p),
                ("overwrite", c_int32)]


class OutputsC(ctypes.Structure):
    _fields_ = [("color", c_void_p), ("raw", c_void_p), ("alpha", c_void_p),
                ("transmittance", c_void_p), ("depth", c_void_p), ("pixel_count", c_void_p),
                ("contributions", c_void_p), ("defer_contributions", c_int32)]


BSR_MAX_GROUPS = 16


class LayoutC(ctypes.Structure):
    _fields_ = [("n", c_int64), ("n_groups", c_int32), ("width", c_int32 * BSR_MAX_GROUPS),
                ("start", c_int64 * BSR_MAX_GROUPS), ("g_positions", c_int32), ("g_rotations", c_int32),
                ("g_log_scales", c_int32), ("g_opacity", c_int32)]


class LrScheduleC(ctypes.Structure):
    _fields_ = [("lr_init", c_double), ("lr_final", c_double), ("max_steps", c_int64),
                ("delay_steps", c_int64), ("delay_mult", c_double), ("scale", c_double)]


class ProfileC(ctypes.Structure):
    _fields_ = [("stats", c_void_p), ("events", c_void_p * 8)]


class FrameInfoC(ctypes.Structure):
    _fields_ = [("visible", c_int64), ("entries", c_int64), ("entries_needed", c_int64),
                ("flagged_pixels", c_int64), ("status", c_int32), ("reserved", c_int32)]


EXPORTS = {
    "bsr_version": (c_int32, [c_void_p, c_void_p]),
    "bsr_status_string": (ctypes.c_char_p, [c_int32]),
    "bsr_frame_bytes": (c_int32, [c_int64, c_int32, c_int32, c_int64, c_void_p]),
    "bsr_forward": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_int64, c_void_p,
                              c_void_p, c_void_p]),
    "bsr_frame_status": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "bsr_contributions": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_int64, c_void_p,
                                    c_void_p]),
    "bsr_view_colors": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p]),
    "bsr_frame_snapshot_bytes": (c_int32, [c_void_p]),
    "bsr_frame_status_async": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "bsr_frame_snapshot_decode": (c_int32, [c_void_p, c_void_p]),
    "bsr_backward": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_int64, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "bsr_backward_deferred_color": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_int64,
                                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                              c_void_p]),
    "bsr_det_workspace_bytes": (c_int32, [c_int64, c_void_p]),
    "bsr_backward_deterministic": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_int64, c_void_p,
                                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_uint64,
                                             c_void_p]),
    "bsr_color_grad_views": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p]),
    "bsr_core_scratch_bytes": (c_int32, [c_int64, c_int32, c_int32, c_int64, c_void_p]),
    "bsr_core_forward_tiled": (c_int32, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_int32, c_int32, c_void_p, c_int32, c_void_p,
                                         c_void_p, c_int64, c_double, c_double, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]),
    "bsr_core_backward": (c_int32, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_int32,
                                    c_void_p, c_void_p, c_int64, c_double, c_double, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_uint64,
                                    c_void_p]),
    "bsr_loss_scratch_bytes": (c_int32, [c_int32, c_int32, c_void_p]),
    "bsr_loss_l1_dssim": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_double,
                                    c_void_p, c_void_p, c_void_p, c_uint64, c_void_p]),
    "bsr_debug_export": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_int64, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p]),
    "bsr_adam_step": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_void_p,
                                c_void_p, c_int64, c_double, c_double, c_double, c_void_p]),
    "bsr_adam_step_device": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_void_p,
                                       c_void_p, c_void_p, c_double, c_double, c_double, c_void_p]),
    "bsr_adam_step_scheduled": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_double,
                                          c_double, c_double, c_void_p]),
    "bsr_codec_scratch_bytes": (c_uint64, [c_int64]),
    "bsr_codec_sort": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_uint64, c_void_p]),
    "bsr_codec_encode": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int32, c_int32,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_void_p]),
    "bsr_codec_decode": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_int32,
                                   c_int32, c_void_p, c_void_p, c_void_p]),
    "bsr_adam_step_fused": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_int32, c_double, c_double, c_double,
                                      c_int32, c_void_p]),
    "bsr_scheduled_lr": (c_double, [c_void_p, c_int64]),
    "bsr_regularizers": (c_int32, [c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p, c_void_p]),
    "bsr_inject_noise": (c_int32, [c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p, c_void_p,
                                   c_uint64, c_uint64, c_void_p, c_void_p]),
    "bsr_mcmc_scratch_bytes": (c_int32, [c_int64, c_void_p]),
    "bsr_find_dead": (c_int32, [c_void_p, c_int64, c_double, c_void_p, c_void_p, c_void_p, c_uint64,
                                c_void_p]),
    "bsr_sample_live": (c_int32, [c_void_p, c_int64, c_double, c_void_p, c_void_p, c_int64, c_void_p,
                                  c_int64, c_void_p, c_uint64, c_uint64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_uint64, c_void_p]),
    "bsr_apply_relocation": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_int64, c_void_p, c_double, c_void_p]),
    "bsr_checkpoint_unpack": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "bsr_checkpoint_pack": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "bsr_grow": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                           c_void_p, c_int64, c_void_p, c_double, c_void_p]),
}

_LIB = None


def load():
    """Load libbsr.so (raises loudly if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libbsr.so not built ({LIB_PATH}); run "
                               "`make -C paper_2501_18630_b200/csrc` or __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def check(status: int, what: str = "libbsr"):
    if status == BSR_OK:
        return
    msg = load().bsr_status_string(status).decode()
    if status == BSR_ERR_DEGENERATE_QUAT:
        raise DegenerateQuaternionError("quaternion norm below 1e-12")
    if status in (BSR_ERR_BAD_ARG, BSR_ERR_FRAME_TOO_SMALL):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (status {status})")


def camera_c(cam) -> CameraC:
    c = CameraC()
    m = [float(v) for v in cam.world_to_camera.reshape(-1)]
    c.world_to_camera = (c_double * 16)(*m)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_18630_b200 needs a CUDA device (no CPU fallback)")
    load()


def stream_ptr():
    """Raw cudaStream_t of torch's current stream on the current device, as a ctypes
    pointer.  Through the C++ accessor: torch.cuda.current_stream() re-runs Python device
    availability checks on every call (~10 us, several times per rendered view)."""
    import torch

    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))
