"""Checkpoints straight into device tensors (mirror of betasplat.sceneio's checkpoint API,
sceneio.py:467-564; format in the reference's docs/formats.md).

The file is the reference's binary little-endian PLY: header comments
``betasplat_checkpoint 1`` and ``lobes M``, one ``double`` property per scalar.  The host
only parses the header and moves the record block; the per-scalar (de)interleave between
the (N, P) fp64 records and the flat group-major fp32 parameter buffer runs on the device
(libbsr ``bsr_checkpoint_unpack`` / ``bsr_checkpoint_pack``).

* ``load_checkpoint(path)`` -> device ``PrimitiveSet`` (fp32; values rounded once).
* ``save_checkpoint(path, prims)`` writes exactly the bytes the reference's
  ``save_checkpoint`` writes for the same (fp32-valued) parameters, so the reference's
  ``load_checkpoint`` reads it, and save -> load round-trips bit-exactly.
* SH-colour sets (the BASELINE configs) use the same container with a ``sh_coeffs K``
  comment instead of ``lobes`` and properties ``sh{k}_r sh{k}_g sh{k}_b`` after ``shape``
  (an extension: the reference has no SH checkpoints).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .primitive import PrimitiveSet, group_layout, group_widths

CHECKPOINT_VERSION = 1  # sceneio.py CHECKPOINT_VERSION
_PLY_TYPES = {"char": "i1", "uchar": "u1", "short": "i2", "ushort": "u2", "int": "i4", "uint": "u4",
              "float": "f4", "double": "f8", "int8": "i1", "uint8": "u1", "int16": "i2", "uint16": "u2",
              "int32": "i4", "uint32": "u4", "float32": "f4", "float64": "f8"}


class CheckpointError(ValueError):
    """sceneio.py:35-36."""


def checkpoint_properties(lobes: int | None = None, sh_coeffs: int | None = None):
    """[(property name, group, component)] in file order (sceneio.py:467-477)."""
    props = [("x", "positions", 0), ("y", "positions", 1), ("z", "positions", 2), ("opacity_raw", "opacity_raw", 0)]
    props += [(f"log_scale_{a}", "log_scales", i) for i, a in enumerate("xyz")]
    props += [(f"rot_{a}", "rotations", i) for i, a in enumerate("wxyz")]
    props += [("shape", "shapes", 0)]
    if sh_coeffs is not None:
        for k in range(sh_coeffs):
            props += [(f"sh{k}_{c}", "sh", 3 * k + i) for i, c in enumerate("rgb")]
        return props
    props += [(f"base_{c}", "base_colors", i) for i, c in enumerate("rgb")]
    for m in range(lobes):
        props += [(f"lobe{m}_axis_{a}", "lobe_axes", 3 * m + i) for i, a in enumerate("xyz")]
        props += [(f"lobe{m}_{c}", "lobe_colors", 3 * m + i) for i, c in enumerate("rgb")]
    return props


def _tables(n, lobes, sh_coeffs):
    layout, _ = group_layout(n, sh_coeffs, None if sh_coeffs is not None else lobes)
    start = {g: a for g, a, _, _ in layout}
    widths = group_widths(sh_coeffs, None if sh_coeffs is not None else lobes)
    props = checkpoint_properties(lobes, sh_coeffs)
    st = (ctypes.c_int64 * len(props))(*[start[g] + c for _, g, c in props])
    sd = (ctypes.c_int32 * len(props))(*[widths[g] for _, g, _ in props])
    return props, st, sd


def _stream():
    return _lib.stream_ptr()


def _parse_header(fh):
    """sceneio.py:288-317: binary little-endian only, no list properties."""
    if fh.readline().strip() != b"ply":
        raise CheckpointError("not a PLY file")
    fmt, comments, elements = None, [], []
    while True:
        line = fh.readline()
        if not line:
            raise CheckpointError("unterminated PLY header")
        tok = line.decode("ascii", "replace").strip().split()
        if not tok:
            continue
        if tok[0] == "format":
            fmt = tok[1]
        elif tok[0] == "comment":
            comments.append(" ".join(tok[1:]))
        elif tok[0] == "element":
            elements.append((tok[1], int(tok[2]), []))
        elif tok[0] == "property":
            if tok[1] == "list":
                raise CheckpointError("list properties are not supported")
            if tok[1] not in _PLY_TYPES:
                raise CheckpointError(f"unknown PLY type {tok[1]}")
            elements[-1][2].append((tok[2], "<" + _PLY_TYPES[tok[1]]))
        elif tok[0] == "end_header":
            break
    if fmt != "binary_little_endian":
        raise CheckpointError(f"unsupported PLY format {fmt!r} (need binary_little_endian)")
    return comments, elements


def load_checkpoint(path, device="cuda") -> PrimitiveSet:
    """sceneio.load_checkpoint (sceneio.py:514-564) into a device PrimitiveSet."""
    with open(path, "rb") as fh:
        comments, elements = _parse_header(fh)
        vertex = next((e for e in elements if e[0] == "vertex"), None)
        if vertex is None:
            raise CheckpointError(f"{path}: no vertex element")
        _, n, props = vertex
        raw = fh.read()
    version = lobes = shk = None
    for c in comments:
        parts = c.split()
        if parts[:1] == ["betasplat_checkpoint"]:
            version = int(parts[1])
        elif parts[:1] == ["lobes"]:
            lobes = int(parts[1])
        elif parts[:1] == ["sh_coeffs"]:
            shk = int(parts[1])
    if version is None:
        raise CheckpointError(f"{path}: not a betasplat checkpoint")
    if version != CHECKPOINT_VERSION:
        raise CheckpointError(f"{path}: unsupported checkpoint version {version}")
    if lobes is None and shk is None:
        raise CheckpointError(f"{path}: missing lobe count")
    names, st, sd = _tables(n, lobes, shk)
    if [p[0] for p in props] != [p[0] for p in names] or any(t != "<f8" for _, t in props):
        raise CheckpointError(f"{path}: property list does not match {lobes} lobes")
    nbytes = n * len(names) * 8
    if len(raw) < nbytes:
        raise CheckpointError(f"{path}: truncated vertex data")
    _lib.require_cuda()
    host = torch.frombuffer(bytearray(raw[:nbytes]), dtype=torch.float64) if nbytes else torch.zeros(0, dtype=torch.float64)
    rec = (torch.empty(host.shape, dtype=host.dtype, pin_memory=True).copy_(host).to(device, non_blocking=True)
           if nbytes else host.to(device))
    _, total = group_layout(n, shk, None if shk is not None else lobes)
    flat = torch.zeros(total, dtype=torch.float32, device=device)
    _lib.check(_lib.load().bsr_checkpoint_unpack(rec.data_ptr() if nbytes else None, n, len(names), st, sd,
                                                  flat.data_ptr(), _stream()), "load_checkpoint")
    return PrimitiveSet.from_flat(n, shk, flat, None if shk is not None else lobes)


def save_checkpoint(path, prims: PrimitiveSet):
    """sceneio.save_checkpoint (sceneio.py:480-511): same header and record bytes."""
    _lib.require_cuda()
    n = len(prims)
    sh = prims.color_model == "sh"
    names, st, sd = _tables(n, prims.lobes, prims.k if sh else None)
    rec = torch.empty(max(n * len(names), 1), dtype=torch.float64, device=prims.flat.device)
    _lib.check(_lib.load().bsr_checkpoint_pack(prims.flat.data_ptr(), n, len(names), st, sd, rec.data_ptr(),
                                                _stream()), "save_checkpoint")
    header = ["ply", "format binary_little_endian 1.0", f"comment betasplat_checkpoint {CHECKPOINT_VERSION}",
              f"comment sh_coeffs {prims.k}" if sh else f"comment lobes {prims.lobes}", f"element vertex {n}"]
    header += [f"property double {name}" for name, _, _ in names]
    header.append("end_header")
    data = rec[: n * len(names)].cpu().numpy().astype("<f8", copy=False)
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        fh.write(data.tobytes())


__all__ = ["CHECKPOINT_VERSION", "CheckpointError", "checkpoint_properties", "load_checkpoint", "save_checkpoint"]
