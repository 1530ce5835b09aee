"""Post-training codec with the byte work on the device (mirror of betasplat.compression,
compression.py:1-258; archive layout in the reference's docs/formats.md).

``pack(prims, out_dir, sort=True)`` writes the reference's archive -- ``manifest.json``
plus one 8-bit PNG per attribute group and four position byte-plane PNGs -- byte for byte
(same arrays, same OpenCV PNG call); ``unpack(archive_dir)`` reads it back into a device
``PrimitiveSet``.  On the device (libbsr ``bsr_codec_*``): Morton keys and their stable
sort, per-channel min / max, 8-bit quantisation into the padded grids, the position byte
planes, and the inverse.  The host parses the manifest and runs the PNG codec.

Spherical-Beta sets use the reference's groups exactly.  SH-colour sets (the BASELINE
configs) use the same container with an ``sh_coeffs`` manifest key and one RGB group per
coefficient (``sh{k}``) in place of ``base_colors`` / lobes -- an extension, the
reference has no SH archives.

Differences: quantisation is fixed at 8 bits (the reference's QUANT_BITS; its
``quantize_attribute(bits > 8)`` helper has no device counterpart), and decoded
attributes are fp32 (the reference returns fp64; decode computes in fp64 and rounds
once).
"""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np
import torch

from . import _lib
from .primitive import PrimitiveSet, group_layout

ARCHIVE_VERSION = 1  # compression.py:24
QUANT_BITS = 8
PNG_LEVEL = 9


class ArchiveError(ValueError):
    """compression.py:30-31."""


class CodecGroupC(ctypes.Structure):
    _fields_ = [("start", ctypes.c_int64), ("stride", ctypes.c_int32), ("channels", ctypes.c_int32)]


def _stream():
    return _lib.stream_ptr()


# ----------------------------------------------------------------------------- PNG I/O
def write_png(path, array, compression=6):
    """sceneio.write_png (sceneio.py:61-74): uint8/uint16 gray, RGB or RGBA via OpenCV."""
    import cv2

    array = np.asarray(array)
    if array.dtype not in (np.uint8, np.uint16):
        raise ValueError("write_png stores uint8 or uint16 samples")
    if array.ndim == 3 and array.shape[2] == 3:
        array = array[:, :, ::-1]
    elif array.ndim == 3 and array.shape[2] == 4:
        array = array[:, :, [2, 1, 0, 3]]
    elif array.ndim != 2:
        raise ValueError(f"unsupported image shape {array.shape}")
    if not cv2.imwrite(str(path), np.ascontiguousarray(array), [cv2.IMWRITE_PNG_COMPRESSION, compression]):
        raise IOError(f"failed to write PNG {path}")


def read_png(path):
    """sceneio.read_png (sceneio.py:77-90)."""
    import cv2

    with open(path, "rb") as fh:
        if fh.read(8)[:4] != b"\x89PNG":
            raise IOError(f"{path} is not a PNG file")
    arr = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    if arr is None:
        raise IOError(f"failed to decode PNG {path}")
    if arr.ndim == 3 and arr.shape[2] == 3:
        arr = arr[:, :, ::-1]
    elif arr.ndim == 3 and arr.shape[2] == 4:
        arr = arr[:, :, [2, 1, 0, 3]]
    return np.ascontiguousarray(arr)


# ----------------------------------------------------------------------------- layout
def grid_dims(count):
    """compression.py:106-109."""
    count = max(int(count), 1)
    cols = int(np.ceil(np.sqrt(count)))
    return int(np.ceil(count / cols)), cols


def attribute_groups(n, k=None, lobes=None):
    """[(name, flat start, stride, channels)] in archive order (compression.py:125-138)."""
    layout, _ = group_layout(n, k, lobes)
    start = {g: a for g, a, _, _ in layout}
    out = [("opacity_raw", start["opacity_raw"], 1, 1), ("log_scales", start["log_scales"], 3, 3),
           ("rotations", start["rotations"], 4, 4), ("shapes", start["shapes"], 1, 1)]
    if lobes is None:
        out += [(f"sh{c}", start["sh"] + 3 * c, 3 * k, 3) for c in range(k)]
    else:
        out.append(("base_colors", start["base_colors"], 3, 3))
        for m in range(lobes):
            out.append((f"lobe{m}_axes", start["lobe_axes"] + 3 * m, 3 * lobes, 3))
            out.append((f"lobe{m}_colors", start["lobe_colors"] + 3 * m, 3 * lobes, 3))
    return out


def _groups_c(groups):
    arr = (CodecGroupC * max(len(groups), 1))()
    for i, (_, s, st, c) in enumerate(groups):
        arr[i].start, arr[i].stride, arr[i].channels = s, st, c
    return arr


def _scratch(n, device):
    nbytes = int(_lib.load().bsr_codec_scratch_bytes(n))
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device), nbytes


# ----------------------------------------------------------------------------- keys / sort
def morton_keys(positions) -> torch.Tensor:
    """compression.morton_keys (compression.py:45-59) on the device: uint64 keys as int64."""
    _lib.require_cuda()
    pos = torch.as_tensor(positions, dtype=torch.float32, device="cuda").contiguous()
    n = pos.shape[0]
    keys = torch.empty(n, dtype=torch.int64, device=pos.device)
    perm = torch.empty(n, dtype=torch.int64, device=pos.device)
    if n:
        scratch, nbytes = _scratch(n, pos.device)
        _lib.check(_lib.load().bsr_codec_sort(pos.data_ptr(), n, keys.data_ptr(), perm.data_ptr(),
                                              scratch.data_ptr(), nbytes, _stream()), "morton_keys")
    return keys


def sort_primitives(prims: PrimitiveSet) -> torch.Tensor:
    """compression.sort_primitives (compression.py:62-66): the stable Morton permutation."""
    _lib.require_cuda()
    n = len(prims)
    perm = torch.empty(n, dtype=torch.int64, device=prims.flat.device)
    if n:
        scratch, nbytes = _scratch(n, prims.flat.device)
        pos = prims.positions
        _lib.check(_lib.load().bsr_codec_sort(pos.data_ptr(), n, None, perm.data_ptr(), scratch.data_ptr(), nbytes,
                                              _stream()), "sort_primitives")
    return perm


# ----------------------------------------------------------------------------- pack / unpack
def encode(prims: PrimitiveSet, sort=True):
    """Device half of pack: (perm or None, rows, cols, planes (4, rows, cols, 3) uint8,
    {group: codes (rows, cols[, C]) uint8}, {group: (mins, maxs)}) -- host numpy arrays."""
    _lib.require_cuda()
    n = len(prims)
    if n == 0:
        raise ValueError("zero-size array to reduction operation minimum which has no identity")
    dev = prims.flat.device
    rows, cols = grid_dims(n)
    cells = rows * cols
    sh = prims.color_model == "sh"
    groups = attribute_groups(n, prims.k if sh else None, None if sh else prims.lobes)
    lib = _lib.load()
    scratch, nbytes = _scratch(n, dev)
    perm = None
    if sort:
        perm = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(lib.bsr_codec_sort(prims.positions.data_ptr(), n, None, perm.data_ptr(), scratch.data_ptr(),
                                      nbytes, _stream()), "pack")
    channels = sum(g[3] for g in groups)
    planes = torch.empty((4, cells, 3), dtype=torch.uint8, device=dev)
    codes = torch.empty(cells * channels, dtype=torch.uint8, device=dev)
    mm = torch.empty((2, channels), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.bsr_codec_encode(prims.flat.data_ptr(), prims.positions.data_ptr(), n,
                                    _lib.ptr(perm), len(groups), _groups_c(groups), rows, cols,
                                    planes.data_ptr(), codes.data_ptr(), mm[0].data_ptr(), mm[1].data_ptr(),
                                    status.data_ptr(), scratch.data_ptr(), nbytes, _stream()), "pack")
    # one device->host copy of everything the PNG encoder and the manifest need
    host = torch.cat([status.view(torch.uint8), mm.view(-1).view(torch.uint8), planes.view(-1), codes]).cpu().numpy()
    if int(host[:4].view(np.int32)[0]) != 0:
        raise ValueError("cannot quantize non-finite values")
    o = 4
    mmh = host[o:o + 16 * channels].view(np.float64).reshape(2, channels)
    o += 16 * channels
    pl = host[o:o + 12 * cells].reshape(4, rows, cols, 3)
    o += 12 * cells
    out_codes, ranges, c0 = {}, {}, 0
    for name, _, _, c in groups:
        g = host[o:o + cells * c].reshape(rows, cols, c)
        out_codes[name] = g[:, :, 0] if c == 1 else g
        ranges[name] = (mmh[0, c0:c0 + c].copy(), mmh[1, c0:c0 + c].copy())
        o += cells * c
        c0 += c
    return perm, rows, cols, pl, out_codes, ranges


def pack(prims: PrimitiveSet, out_dir, sort=True):
    """compression.pack (compression.py:141-187); returns the manifest."""
    os.makedirs(out_dir, exist_ok=True)
    _, rows, cols, planes, codes, ranges = encode(prims, sort)
    sh = prims.color_model == "sh"
    manifest = {"version": ARCHIVE_VERSION, "count": len(prims), "lobes": 0 if sh else prims.lobes,
                "grid": [rows, cols], "order": "morton" if sort else "keep", "quant_bits": QUANT_BITS,
                "attributes": {}, "position_planes": []}
    if sh:
        manifest["sh_coeffs"] = prims.k
    jobs = []
    for b in range(4):
        name = f"positions_byte{b}.png"
        jobs.append((os.path.join(out_dir, name), planes[b]))
        manifest["position_planes"].append(name)
    for name, grid in codes.items():
        fn = f"{name}.png"
        jobs.append((os.path.join(out_dir, fn), grid))
        mins, maxs = ranges[name]
        manifest["attributes"][name] = {"file": fn, "channels": 1 if grid.ndim == 2 else int(grid.shape[2]),
                                        "min": [float(v) for v in mins], "max": [float(v) for v in maxs]}
    # the PNGs are independent deflate streams: encode them concurrently (OpenCV releases
    # the GIL); the bytes are those of the serial loop
    _parallel(lambda j: write_png(j[0], j[1], PNG_LEVEL), jobs)
    with open(os.path.join(out_dir, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    return manifest


def _parallel(fn, items):
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(items), os.cpu_count() or 1) or 1) as ex:
        return list(ex.map(fn, items))


def unpack(archive_dir, device="cuda") -> PrimitiveSet:
    """compression.unpack (compression.py:190-250) into a device PrimitiveSet (fp32)."""
    path = os.path.join(archive_dir, "manifest.json")
    if not os.path.exists(path):
        raise ArchiveError(f"no manifest at {path}")
    with open(path) as fh:
        manifest = json.load(fh)
    if manifest.get("version") != ARCHIVE_VERSION:
        raise ArchiveError(f"unsupported archive version {manifest.get('version')}")
    n, rows, cols = int(manifest["count"]), *[int(v) for v in manifest["grid"]]
    if rows * cols < n:
        raise ArchiveError("grid smaller than primitive count")
    shk = manifest.get("sh_coeffs")
    lobes = None if shk is not None else int(manifest["lobes"])
    cells = rows * cols
    groups = attribute_groups(n, shk, lobes)
    specs = []
    for name, _, _, c in groups:
        spec = manifest["attributes"].get(name)
        if spec is None:
            raise ArchiveError(f"manifest missing attribute {name}")
        specs.append(spec)
    files = list(manifest["position_planes"]) + [spec["file"] for spec in specs]
    images = _parallel(lambda f: read_png(os.path.join(archive_dir, f)), files)
    planes = []
    for name, g in zip(manifest["position_planes"], images):
        if g.shape[:2] != (rows, cols) or g.dtype != np.uint8:
            raise ArchiveError(f"{name}: unexpected plane shape or depth")
        if g.ndim != 3 or g.shape[2] != 3:
            raise ArchiveError(f"{name}: expected an RGB byte plane")
        planes.append(g)
    if len(planes) != 4:
        raise ArchiveError("expected four position byte planes")
    blobs, mins, maxs = [np.stack(planes).reshape(-1)], [], []
    for (name, _, _, c), spec, g in zip(groups, specs, images[len(manifest["position_planes"]):]):
        got = 1 if g.ndim == 2 else g.shape[2]
        if got != spec["channels"] or spec["channels"] != c:
            raise ArchiveError(f"{name}: channel count mismatch")
        if g.shape[:2] != (rows, cols) or g.dtype != np.uint8:
            raise ArchiveError(f"{name}: unexpected grid shape or depth")
        blobs.append(g.reshape(-1))
        mins += list(spec["min"])
        maxs += list(spec["max"])
    _lib.require_cuda()
    # one host->device copy: [mins, maxs (fp64)] [planes] [codes]
    host = np.concatenate([np.asarray(mins + maxs, np.float64).view(np.uint8)] + blobs)
    dev = torch.from_numpy(host).pin_memory().to(device, non_blocking=True)
    nb_mm, nb_planes = 16 * len(mins), 12 * cells
    nb_codes = host.size - nb_mm - nb_planes
    mm = dev[:nb_mm].view(torch.float64)
    planes_d = dev[nb_mm:nb_mm + nb_planes]
    codes_d = dev[nb_mm + nb_planes:]
    _, total = group_layout(n, shk, lobes)
    flat = torch.zeros(total, dtype=torch.float32, device=device)
    prims = PrimitiveSet.from_flat(n, shk, flat, lobes)
    ch = len(mins)
    _lib.check(_lib.load().bsr_codec_decode(planes_d.data_ptr(), codes_d.data_ptr() if nb_codes else None,
                                            mm[:ch].data_ptr() if ch else None, mm[ch:].data_ptr() if ch else None,
                                            n, len(groups), _groups_c(groups), rows, cols, flat.data_ptr(),
                                            prims.positions.data_ptr(), _stream()), "unpack")
    return prims


def archive_size(archive_dir):
    """compression.py:253-257."""
    return sum(os.path.getsize(os.path.join(archive_dir, f)) for f in os.listdir(archive_dir))


__all__ = ["ARCHIVE_VERSION", "QUANT_BITS", "PNG_LEVEL", "ArchiveError", "archive_size", "attribute_groups", "encode",
           "grid_dims", "morton_keys", "pack", "read_png", "sort_primitives", "unpack", "write_png"]
