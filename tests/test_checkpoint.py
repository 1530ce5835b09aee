"""Checkpoint I/O (sceneio.py:467-564): reference-written PLY files (tests/golden/ckpt_*.ply,
made by the reference's own save_checkpoint from fp32-valued parameters) load into device
tensors exactly, and save_checkpoint reproduces the reference's bytes."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

SB = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "base_colors", "lobe_axes", "lobe_colors")


def _read_reference_ply(path):
    """Independent host decode of the golden file (header + structured record array)."""
    with open(path, "rb") as fh:
        head = []
        while True:
            line = fh.readline().decode().strip()
            head.append(line)
            if line == "end_header":
                break
        names = [l.split()[2] for l in head if l.startswith("property")]
        n = int(next(l for l in head if l.startswith("element vertex")).split()[2])
        rec = np.frombuffer(fh.read(), dtype=np.dtype([(nm, "<f8") for nm in names]), count=n)
    return head, rec


def _bad(tmp_path, text, payload=b""):
    p = tmp_path / "bad.ply"
    p.write_bytes(text.encode() + payload)
    return str(p)


def test_header_errors_match_reference(tmp_path):
    from paper_2501_18630_b200.sceneio import CheckpointError, load_checkpoint

    with pytest.raises(CheckpointError, match="not a PLY"):
        load_checkpoint(_bad(tmp_path, "plx\n"))
    with pytest.raises(CheckpointError, match="unsupported PLY format"):
        load_checkpoint(_bad(tmp_path, "ply\nformat ascii 1.0\nend_header\n"))
    with pytest.raises(CheckpointError, match="not a betasplat checkpoint"):
        load_checkpoint(_bad(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 0\nend_header\n"))
    with pytest.raises(CheckpointError, match="unsupported checkpoint version"):
        load_checkpoint(_bad(tmp_path, "ply\nformat binary_little_endian 1.0\ncomment betasplat_checkpoint 2\n"
                                       "comment lobes 0\nelement vertex 0\nend_header\n"))
    with pytest.raises(CheckpointError, match="does not match"):
        load_checkpoint(_bad(tmp_path, "ply\nformat binary_little_endian 1.0\ncomment betasplat_checkpoint 1\n"
                                       "comment lobes 1\nelement vertex 0\nproperty double x\nend_header\n"))
    with pytest.raises(CheckpointError, match="list properties"):
        load_checkpoint(_bad(tmp_path, "ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                                       "property list uchar int idx\nend_header\n"))


def test_property_order_matches_reference_file():
    from paper_2501_18630_b200.sceneio import checkpoint_properties

    for name, lobes in (("ckpt_l2.ply", 2), ("ckpt_l0.ply", 0)):
        head, _ = _read_reference_ply(os.path.join(GOLDEN, name))
        assert [l.split()[2] for l in head if l.startswith("property")] == [p[0] for p in checkpoint_properties(lobes)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,lobes", [("ckpt_l2.ply", 2), ("ckpt_l0.ply", 0)])
def test_reference_checkpoint_roundtrip(name, lobes, tmp_path, cuda):
    from paper_2501_18630_b200.sceneio import load_checkpoint, save_checkpoint

    path = os.path.join(GOLDEN, name)
    _, rec = _read_reference_ply(path)
    prims = load_checkpoint(path)
    assert len(prims) == rec.shape[0] and prims.lobes == lobes
    np.testing.assert_array_equal(prims.positions.cpu().numpy(), np.stack([rec["x"], rec["y"], rec["z"]], -1))
    np.testing.assert_array_equal(prims.rotations.cpu().numpy(), np.stack([rec[f"rot_{a}"] for a in "wxyz"], -1))
    np.testing.assert_array_equal(prims.opacity_raw.cpu().numpy(), rec["opacity_raw"])
    np.testing.assert_array_equal(prims.shapes.cpu().numpy(), rec["shape"])
    if lobes:
        np.testing.assert_array_equal(prims.lobe_colors[:, 1, 2].cpu().numpy(), rec["lobe1_b"])
    out = tmp_path / "ours.ply"
    save_checkpoint(str(out), prims)
    assert out.read_bytes() == open(path, "rb").read()  # the reference's exact bytes


@pytest.mark.gpu
def test_sh_checkpoint_roundtrip(tmp_path, cuda):
    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.scenes import make_workload
    from paper_2501_18630_b200.sceneio import load_checkpoint, save_checkpoint

    wl = make_workload("c1", seed=2, n=300, width=64, height=64)
    a = PrimitiveSet.from_scene(wl.scene)
    save_checkpoint(str(tmp_path / "sh.ply"), a)
    b = load_checkpoint(str(tmp_path / "sh.ply"))
    assert b.sh_coeffs == 16 and len(b) == 300
    import torch

    assert torch.equal(a.flat, b.flat)
