"""CPU-only checks of the host side: the C-ABI library loads and exports every symbol
include/bsr.h declares, host-side validation, workload generators, layouts."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO


def _header_symbols():
    txt = open(os.path.join(REPO, "include", "bsr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|size_t|const char \*)\s*(bsr_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2501_18630_b200 import _lib

    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.EXPORTS, f"{s} has no ctypes signature"


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {os.path.join(REPO, 'paper_2501_18630_b200', 'libbsr.so')} 2>&1").read()
    assert "sm_100a" in out


def test_host_side_validation_without_gpu():
    from paper_2501_18630_b200 import _lib

    lib = _lib.load()
    out = ctypes.c_uint64()
    assert lib.bsr_frame_bytes(1000, 64, 64, 5000, ctypes.byref(out)) == 0 and out.value > 0
    assert lib.bsr_frame_bytes(-1, 64, 64, 10, ctypes.byref(out)) == _lib.BSR_ERR_BAD_ARG
    assert lib.bsr_frame_bytes(10, 0, 64, 10, ctypes.byref(out)) == _lib.BSR_ERR_BAD_ARG
    assert lib.bsr_loss_scratch_bytes(10, 10, ctypes.byref(out)) == _lib.BSR_ERR_BAD_ARG
    assert lib.bsr_status_string(2) == b"tile-entry capacity exceeded"
    with pytest.raises(ValueError):
        _lib.check(_lib.BSR_ERR_BAD_ARG)
    with pytest.raises(_lib.DegenerateQuaternionError):
        _lib.check(_lib.BSR_ERR_DEGENERATE_QUAT)
    # bad scene descriptor is rejected before any device work
    sc = _lib.SceneC()
    sc.n, sc.sh_coeffs = 5, 7
    cam = _lib.CameraC()
    cam.width, cam.height, cam.fx, cam.fy = 8, 8, 1.0, 1.0
    bg = (ctypes.c_float * 3)(1, 1, 1)
    o = _lib.OutputsC()
    assert lib.bsr_forward(ctypes.byref(sc), ctypes.byref(cam), bg, ctypes.c_void_p(1), 1, 10,
                           ctypes.byref(o), None, None) == _lib.BSR_ERR_BAD_ARG


def test_frame_bytes_monotone_in_capacity():
    from paper_2501_18630_b200 import _lib

    lib = _lib.load()
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    lib.bsr_frame_bytes(100_000, 800, 800, 400_000, ctypes.byref(a))
    lib.bsr_frame_bytes(100_000, 800, 800, 800_000, ctypes.byref(b))
    assert b.value > a.value


def test_camera_conventions_match_reference():
    """primitive.py:123-137: fx from horizontal fov, principal point ((W-1)/2, (H-1)/2)."""
    from paper_2501_18630_b200.camera import Camera

    cam = Camera.from_lookat((0, 0, 4), (0, 0, 0), (0, 1, 0), np.deg2rad(60), 256, 256)
    assert cam.fx == pytest.approx(221.70250336881628)
    assert cam.cx == 127.5 and cam.cy == 127.5
    np.testing.assert_allclose(cam.center, [0, 0, 4], atol=1e-12)
    with pytest.raises(ValueError):
        Camera(np.eye(3), 1, 1, 0, 0, 4, 4)
    with pytest.raises(ValueError):
        Camera(np.diag([1.0, 2, 1, 1]), 1, 1, 0, 0, 4, 4)


def test_workloads_are_seeded_and_fp32():
    from paper_2501_18630_b200.scenes import make_workload

    a = make_workload("c1", seed=0, n=1000)
    b = make_workload("c1", seed=0, n=1000)
    for k, v in a.scene.arrays().items():
        assert v.dtype == np.float32
        np.testing.assert_array_equal(v, b.scene.arrays()[k])
    assert a.scene.sh.shape == (1000, 16, 3)
    c3 = make_workload("c3", seed=0, n=1000, views=32)
    assert len(c3.cameras) == 32
    for cam in c3.cameras:
        assert cam.center[1] > 0 and np.linalg.norm(cam.center) == pytest.approx(8.0)
    c4 = make_workload("c4", seed=0, n=1000)
    assert c4.cameras[0].width == 3840 and c4.cameras[0].height == 2160


def test_flat_group_layout():
    from paper_2501_18630_b200.primitive import group_layout

    for n in (10, 11, 100_001):
        layout, total = group_layout(n, 16)
        assert total >= n * (3 + 4 + 3 + 1 + 1 + 48)
        names = [g for g, *_ in layout]
        assert names == ["positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"]
        for _, a, b, shape in layout:
            assert (a * 4) % 16 == 0  # float4-aligned group starts
            assert b - a == int(np.prod(shape))


def test_backend_seam_errors():
    from paper_2501_18630_b200 import backend

    with pytest.raises(ValueError):
        backend.get_core("compiled-nope")
