"""The ``cuda`` raster core: the reference's core-plugin seam on the B200.

Same three functions and signatures as betasplat._raster / _raster_py
(_raster.pyx:24-27, 130-134, 244-249): numpy fp64 in, numpy out, inputs already depth
sorted and visible-only.  Internally the arrays go to the device once, the raster runs
in fp32 with fp64 replay of uncertified pixels (libbsr.so), and results come back as
fp64 (images) / int64 (contributions).  ``threads`` is accepted and ignored.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

COMPILED = True
TILE = 16


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def _bins_for_naive(bounds, height, width):
    """forward_naive == tiled compositing over the bounds-derived tile lists (the reference
    asserts the two agree, tests/test_rasterizer.py:150-158); build the lists on the host."""
    tiles_x = (width + TILE - 1) // TILE
    n_tiles = tiles_x * ((height + TILE - 1) // TILE)
    if bounds.shape[0] == 0:
        return np.zeros(n_tiles + 1, np.int64), np.zeros(0, np.int64)
    tx0, tx1 = bounds[:, 0] // TILE, bounds[:, 1] // TILE
    ty0, ty1 = bounds[:, 2] // TILE, bounds[:, 3] // TILE
    sx = (tx1 - tx0 + 1).astype(np.int64)
    counts = sx * (ty1 - ty0 + 1)
    ids = np.repeat(np.arange(bounds.shape[0], dtype=np.int64), counts)
    local = np.arange(int(counts.sum()), dtype=np.int64) - np.repeat(np.cumsum(counts) - counts, counts)
    rsx = np.repeat(sx, counts)
    tile_ids = (np.repeat(ty0, counts) + local // rsx) * tiles_x + np.repeat(tx0, counts) + local % rsx
    lists = ids[np.argsort(tile_ids, kind="stable")]
    offsets = np.zeros(n_tiles + 1, np.int64)
    np.cumsum(np.bincount(tile_ids, minlength=n_tiles), out=offsets[1:])
    return offsets, lists


def _scratch(v, width, height, e):
    out = ctypes.c_uint64()
    _lib.check(_lib.load().bsr_core_scratch_bytes(v, width, height, e, ctypes.byref(out)))
    return torch.empty(int(out.value), dtype=torch.uint8, device="cuda"), int(out.value)


def _stream():
    return _lib.stream_ptr()


def forward_tiled(means, conics, opac, betas, colors, bounds, height, width, background, tile_size,
                  offsets, lists, threads, alpha_min, t_stop, return_extra=False):
    _lib.require_cuda()
    if tile_size != TILE:
        raise ValueError("the cuda core supports tile_size == 16")
    v = int(np.asarray(means).shape[0])
    e = int(np.asarray(lists).shape[0])
    d = [_dev(means, np.float64), _dev(conics, np.float64), _dev(opac, np.float64),
         _dev(betas, np.float64), _dev(colors, np.float64)]
    bd = _dev(bounds, np.int32)
    off, lst = _dev(offsets, np.int64), _dev(lists if e else np.zeros(1), np.int64)
    bg = (ctypes.c_double * 3)(*np.asarray(background, np.float64).reshape(3).tolist())
    raw = torch.empty((height, width, 3), dtype=torch.float32, device="cuda")
    trans = torch.empty((height, width), dtype=torch.float32, device="cuda")
    contrib = torch.zeros(max(v, 1), dtype=torch.int32, device="cuda")
    count = torch.empty((height, width), dtype=torch.int32, device="cuda")
    scratch, nb = _scratch(v, width, height, e)
    flagged = ctypes.c_int64()
    rc = _lib.load().bsr_core_forward_tiled(
        v, *(t.data_ptr() for t in d), bd.data_ptr(), height, width, bg, tile_size, off.data_ptr(),
        lst.data_ptr(), e, float(alpha_min), float(t_stop), raw.data_ptr(), trans.data_ptr(),
        contrib.data_ptr(), count.data_ptr(), scratch.data_ptr(), nb, ctypes.byref(flagged), _stream())
    _lib.check(rc, "core.forward_tiled")
    raw_np = raw.double().cpu().numpy()
    t_np = trans.double().cpu().numpy()
    out = (raw_np, 1.0 - t_np, t_np, contrib[:v].long().cpu().numpy())
    if return_extra:
        return out + (dict(pixel_count=count.cpu().numpy(), flagged=int(flagged.value)),)
    return out


def forward_naive(means, conics, opac, betas, colors, bounds, height, width, background, alpha_min,
                  t_stop):
    offsets, lists = _bins_for_naive(np.asarray(bounds), height, width)
    return forward_tiled(means, conics, opac, betas, colors, bounds, height, width, background, TILE,
                         offsets, lists, 1, alpha_min, t_stop)


def backward(means, conics, opac, betas, colors, bounds, height, width, background, raw, d_raw,
             tile_size, offsets, lists, threads, alpha_min, t_stop):
    _lib.require_cuda()
    if tile_size != TILE:
        raise ValueError("the cuda core supports tile_size == 16")
    v = int(np.asarray(means).shape[0])
    e = int(np.asarray(lists).shape[0])
    d = [_dev(means, np.float64), _dev(conics, np.float64), _dev(opac, np.float64),
         _dev(betas, np.float64), _dev(colors, np.float64)]
    bd = _dev(bounds, np.int32)
    off, lst = _dev(offsets, np.int64), _dev(lists if e else np.zeros(1), np.int64)
    bg = (ctypes.c_double * 3)(*np.asarray(background, np.float64).reshape(3).tolist())
    draw = _dev(d_raw, np.float32)
    vv = max(v, 1)
    dm = torch.zeros((vv, 2), dtype=torch.float32, device="cuda")
    dc = torch.zeros((vv, 3), dtype=torch.float32, device="cuda")
    do = torch.zeros(vv, dtype=torch.float32, device="cuda")
    db = torch.zeros(vv, dtype=torch.float32, device="cuda")
    dcol = torch.zeros((vv, 3), dtype=torch.float32, device="cuda")
    scratch, nb = _scratch(v, width, height, e)
    rc = _lib.load().bsr_core_backward(
        v, *(t.data_ptr() for t in d), bd.data_ptr(), height, width, bg, draw.data_ptr(), tile_size,
        off.data_ptr(), lst.data_ptr(), e, float(alpha_min), float(t_stop), dm.data_ptr(), dc.data_ptr(),
        do.data_ptr(), db.data_ptr(), dcol.data_ptr(), scratch.data_ptr(), nb, _stream())
    _lib.check(rc, "core.backward")
    return tuple(x[:v].double().cpu().numpy() for x in (dm, dc, do, db, dcol))
