"""CPU restatement of the reference's post-training codec (compression.py) -- TEST
INFRASTRUCTURE ONLY: imported by tests/ as the checker for libbsr's bsr_codec_* path,
never by the product.

Pinned against the reference itself: tests/golden/make_golden_train.py `codec` ran the
reference's compression.pack / unpack / morton_keys / sort_primitives on two scenes and
committed the archives (tests/golden/codec_l2, codec_l0_keep) and arrays (codec.npz);
tests/test_codec_oracle.py checks this module against them.

Each function restates the published algorithm in plain numpy (fp64, numpy's round-half-
even) with the reference line it follows.
"""

from __future__ import annotations

import numpy as np

MORTON_BITS = 21
QUANT_LEVELS = 255.0  # QUANT_BITS = 8 (compression.py:26)


def spread21(v):
    """compression.py:34-42: bit i of a 21-bit integer moves to bit 3i (sequential form)."""
    v = np.asarray(v, np.uint64) & np.uint64((1 << MORTON_BITS) - 1)
    out = np.zeros_like(v)
    for i in range(MORTON_BITS):
        out |= ((v >> np.uint64(i)) & np.uint64(1)) << np.uint64(3 * i)
    return out


def morton_keys(positions):
    """compression.py:45-59: per-axis box, 21-bit codes (round half even, clipped),
    interleaved x | y << 1 | z << 2."""
    p = np.asarray(positions, np.float64)
    lo = p.min(axis=0)
    span = p.max(axis=0) - lo
    span = np.where(span == 0.0, 1.0, span)
    top = float((1 << MORTON_BITS) - 1)
    q = np.clip(np.rint((p - lo) / span * top), 0.0, top).astype(np.uint64)
    return spread21(q[:, 0]) | (spread21(q[:, 1]) << np.uint64(1)) | (spread21(q[:, 2]) << np.uint64(2))


def morton_order(positions):
    """compression.py:62-66: stable argsort of the keys."""
    if len(positions) == 0:
        return np.zeros(0, np.int64)
    return np.argsort(morton_keys(positions), kind="stable")


def quantize(values):
    """compression.py:69-90 at 8 bits: (codes uint8, mins, maxs) per channel."""
    flat = np.asarray(values, np.float64).reshape(len(values), -1)
    if not np.isfinite(flat).all():
        raise ValueError("cannot quantize non-finite values")
    mins, maxs = flat.min(axis=0), flat.max(axis=0)
    span = maxs - mins
    safe = np.where(span > 0.0, span, 1.0)
    codes = np.where(span > 0.0, np.rint((flat - mins) / safe * QUANT_LEVELS), 0.0)
    return codes.astype(np.uint8).reshape(np.shape(values)), mins, maxs


def dequantize(codes, mins, maxs):
    """compression.py:93-103: lerp form, exact at the extreme codes."""
    c = np.asarray(codes, np.float64)
    t = c.reshape(len(c), -1) / QUANT_LEVELS
    return (np.asarray(mins) * (1.0 - t) + np.asarray(maxs) * t).reshape(c.shape)


def grid_dims(count):
    """compression.py:106-109: near-square grid, cols = ceil(sqrt(n))."""
    count = max(int(count), 1)
    cols = int(np.ceil(np.sqrt(count)))
    return int(np.ceil(count / cols)), cols


def to_grid(rows_of_values, rows, cols):
    """compression.py:112-117: row-major cells, zero padding; 1 channel -> 2-D."""
    a = np.asarray(rows_of_values)
    a2 = a.reshape(len(a), -1)
    g = np.zeros((rows * cols, a2.shape[1]), a.dtype)
    g[: len(a)] = a2
    g = g.reshape(rows, cols, a2.shape[1])
    return g[:, :, 0] if a2.shape[1] == 1 else g


def position_planes(positions):
    """compression.py:160-166: the four bytes of each fp32 position, byte b -> plane b."""
    bits = np.asarray(positions, np.float32).view(np.uint32)
    return [((bits >> np.uint32(8 * b)) & np.uint32(0xFF)).astype(np.uint8) for b in range(4)]


def planes_to_positions(planes):
    """compression.py:212-218."""
    w = np.zeros(planes[0].shape, np.uint32)
    for b, p in enumerate(planes):
        w |= p.astype(np.uint32) << np.uint32(8 * b)
    return w.view(np.float32).astype(np.float64)
