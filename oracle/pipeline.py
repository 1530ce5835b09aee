"""ORACLE -- test infrastructure only (never imported by the product package).

fp64 numpy restatement of the reference's per-frame pipeline for the hot path, with the
SH-3 colour adapter that SURVEY.md section 8(c) prescribes.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import it,
and only as the checker / CPU baseline.

Every stage cites the reference function it restates (paths relative to
/root/reference/pkg/src/betasplat/):

  sigmoid                 primitive.py:28-35
  quat_to_rotation        primitive.py:48-67
  covariance_many         primitive.py:75-80
  project                 primitive.py:221-277 (+ _pinhole_jacobian :292-299)
  sh_basis / grad         appearance.py:235-261 / :264-300
  depth_order             rasterizer.py:83-85
  tile_bins               rasterizer.py:161-191
  forward                 rasterizer.py:88-141,194-211 with SH colour instead of SB
  backward                rasterizer.py:230-321 with the SH chain (appearance.py:310-318)
  project_backward        primitive.py:302-345, _rotation_grad_to_quat :348-367
  ssim / loss             training.py:36-131
  adam_step               training.py:258-273

Raster cores (the native part):
  core="ref"    the reference's own compiled Cython core, built by oracle/Makefile into
                oracle/_ref/ (no depth, no per-pixel counts)
  core="c"      oracle/raster_oracle.c, our bit-identical restatement (+ depth channel,
                per-pixel counts / last entry / pair counts)
Parity is pinned in tests/test_oracle.py: "c" vs "ref" bit-identical, and this whole
module vs golden vectors produced by the reference package itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os

import numpy as np

ALPHA_MIN = 1.0 / 255.0  # rasterizer.py:28
T_STOP = 1e-4  # rasterizer.py:29
TILE = 16  # rasterizer.py:30
NEAR_PLANE = 0.01  # primitive.py:22
COV_CONDITIONING = 0.3  # primitive.py:24
BOUNDS_GUARD = 1  # primitive.py:25
SHAPE_CLAMP = 10.0  # kernel.py:24
BASE_EXPONENT = 4.0  # kernel.py:25

HERE = os.path.dirname(os.path.abspath(__file__))

_C0 = 0.28209479177387814
_C1 = 0.4886025119029199
_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
       0.5462742152960396)
_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
       -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


# ----------------------------------------------------------------------------- cores
_LIB = None
_REF = None


def c_core():
    """ctypes handle on oracle/libraster_oracle.so (built by ``make -C oracle``)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "libraster_oracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle C core missing: run `make -C {HERE}`")
        lib = ctypes.CDLL(path)
        p = ctypes.c_void_p
        i, i64, d = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        lib.oracle_forward_tiled.argtypes = [i, p, p, p, p, p, p, p, i, i, p, i, p, p, i64, i, d, d,
                                             p, p, p, p, p, p, p]
        lib.oracle_backward.argtypes = [i, p, p, p, p, p, p, p, i, i, p, p, p, p, p, i, p, p, i64, i,
                                        d, d, p, p, p, p, p, p]
        _LIB = lib
    return _LIB


def ref_core():
    """The reference's compiled ``betasplat._raster`` module, built into oracle/_ref/."""
    global _REF
    if _REF is None:
        hits = glob.glob(os.path.join(HERE, "_ref", "_raster*.so"))
        if not hits:
            raise RuntimeError("reference core not built: run `make -C oracle ref` where "
                               "/root/reference exists")
        spec = importlib.util.spec_from_file_location("_raster", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def have_ref_core() -> bool:
    return bool(glob.glob(os.path.join(HERE, "_ref", "_raster*.so")))


def _ptr(a):
    return None if a is None else a.ctypes.data


# ----------------------------------------------------------------------------- geometry
def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def quat_to_rotation(q):
    q = np.asarray(q, dtype=np.float64)
    nrm = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(nrm < 1e-12):
        raise ValueError("quaternion norm below 1e-12")
    w, x, y, z = np.moveaxis(q / nrm, -1, 0)
    r = np.empty(q.shape[:-1] + (3, 3))
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def covariance_many(quats, scales):
    rs = quat_to_rotation(quats) * np.asarray(scales, dtype=np.float64)[..., None, :]
    return rs @ np.swapaxes(rs, -1, -2)


def pinhole_jacobian(t, cam):
    tx, ty, tz = t[:, 0], t[:, 1], t[:, 2]
    jac = np.zeros((t.shape[0], 2, 3))
    jac[:, 0, 0] = cam.fx / tz
    jac[:, 0, 2] = -cam.fx * tx / tz**2
    jac[:, 1, 1] = cam.fy / tz
    jac[:, 1, 2] = -cam.fy * ty / tz**2
    return jac


def project(positions, rotations, scales, cam):
    """EWA projection of the visible subset (primitive.py:221-277)."""
    positions = np.asarray(positions, dtype=np.float64)
    cam_pts = positions @ cam.rotation.T + cam.translation
    idx = np.nonzero(cam_pts[:, 2] > NEAR_PLANE)[0]
    empty = dict(indices=np.zeros(0, np.int64), means2d=np.zeros((0, 2)), cov2d=np.zeros((0, 2, 2)),
                 conics=np.zeros((0, 3)), depths=np.zeros(0), bounds=np.zeros((0, 4), np.int32),
                 cam_points=np.zeros((0, 3)))
    if idx.size == 0:
        return empty
    t = cam_pts[idx]
    tx, ty, tz = t[:, 0], t[:, 1], t[:, 2]
    means = np.stack([cam.fx * tx / tz + cam.cx, cam.fy * ty / tz + cam.cy], axis=-1)
    sigma = covariance_many(np.asarray(rotations, dtype=np.float64)[idx],
                            np.asarray(scales, dtype=np.float64)[idx])
    a = pinhole_jacobian(t, cam) @ cam.rotation
    cov = a @ sigma @ np.swapaxes(a, -1, -2)
    cov[:, 0, 0] += COV_CONDITIONING
    cov[:, 1, 1] += COV_CONDITIONING
    det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] ** 2
    conics = np.stack([cov[:, 1, 1] / det, -cov[:, 0, 1] / det, cov[:, 0, 0] / det], axis=-1)
    ex = np.sqrt(cov[:, 0, 0])
    ey = np.sqrt(cov[:, 1, 1])
    x0 = np.maximum(np.floor(means[:, 0] - ex).astype(np.int32) - BOUNDS_GUARD, 0)
    x1 = np.minimum(np.ceil(means[:, 0] + ex).astype(np.int32) + BOUNDS_GUARD, cam.width - 1)
    y0 = np.maximum(np.floor(means[:, 1] - ey).astype(np.int32) - BOUNDS_GUARD, 0)
    y1 = np.minimum(np.ceil(means[:, 1] + ey).astype(np.int32) + BOUNDS_GUARD, cam.height - 1)
    keep = np.nonzero((x0 <= x1) & (y0 <= y1))[0]
    if keep.size == 0:
        return empty
    return dict(
        indices=idx[keep],
        means2d=np.ascontiguousarray(means[keep]),
        cov2d=np.ascontiguousarray(cov[keep]),
        conics=np.ascontiguousarray(conics[keep]),
        depths=np.ascontiguousarray(tz[keep]),
        bounds=np.ascontiguousarray(np.stack([x0, x1, y0, y1], axis=-1)[keep], dtype=np.int32),
        cam_points=np.ascontiguousarray(t[keep]),
    )


# ----------------------------------------------------------------------------- SH colour
def sh_basis(degree, dirs):
    x, y, z = dirs[..., 0], dirs[..., 1], dirs[..., 2]
    out = [np.full_like(x, _C0)]
    if degree >= 1:
        out += [-_C1 * y, _C1 * z, -_C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        out += [_C2[0] * x * y, _C2[1] * y * z, _C2[2] * (2.0 * zz - xx - yy), _C2[3] * x * z,
                _C2[4] * (xx - yy)]
    if degree >= 3:
        out += [_C3[0] * y * (3.0 * xx - yy), _C3[1] * x * y * z, _C3[2] * y * (4.0 * zz - xx - yy),
                _C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy), _C3[4] * x * (4.0 * zz - xx - yy),
                _C3[5] * z * (xx - yy), _C3[6] * x * (xx - 3.0 * yy)]
    return np.stack(out, axis=-1)


def sh_basis_grad(degree, dirs):
    """d basis / d dir, (..., K, 3)."""
    x, y, z = dirs[..., 0], dirs[..., 1], dirs[..., 2]
    zero = np.zeros_like(x)
    one = np.ones_like(x)

    def v(a, b, c):
        return np.stack([a, b, c], axis=-1)

    out = [v(zero, zero, zero)]
    if degree >= 1:
        out += [v(zero, -_C1 * one, zero), v(zero, zero, _C1 * one), v(-_C1 * one, zero, zero)]
    if degree >= 2:
        out += [_C2[0] * v(y, x, zero), _C2[1] * v(zero, z, y), _C2[2] * v(-2.0 * x, -2.0 * y, 4.0 * z),
                _C2[3] * v(z, zero, x), _C2[4] * v(2.0 * x, -2.0 * y, zero)]
    if degree >= 3:
        xx, yy, zz = x * x, y * y, z * z
        out += [_C3[0] * v(6.0 * x * y, 3.0 * xx - 3.0 * yy, zero),
                _C3[1] * v(y * z, x * z, x * y),
                _C3[2] * v(-2.0 * x * y, 4.0 * zz - xx - 3.0 * yy, 8.0 * y * z),
                _C3[3] * v(-6.0 * x * z, -6.0 * y * z, 6.0 * zz - 3.0 * xx - 3.0 * yy),
                _C3[4] * v(4.0 * zz - 3.0 * xx - yy, -2.0 * x * y, 8.0 * x * z),
                _C3[5] * v(2.0 * x * z, -2.0 * y * z, xx - yy),
                _C3[6] * v(3.0 * xx - 3.0 * yy, -6.0 * x * y, zero)]
    return np.stack(out, axis=-2)


AXIS_EPS = 1e-8  # appearance.py:24


def _effective_axes(axes):
    norms = np.linalg.norm(axes, axis=-1, keepdims=True)
    return np.where(norms < AXIS_EPS, np.array([0.0, 0.0, 1.0]), axes)


def sb_eval_many(base, axes, cols, dirs):
    """appearance.py:108-124: Spherical-Beta colour and lobe responses."""
    ax = _effective_axes(axes)
    norms = np.linalg.norm(ax, axis=-1)
    units = ax / norms[..., None]
    w = np.clip(np.einsum("nmk,nk->nm", units, dirs), 0.0, 1.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        resp = np.where(w > 0.0, w ** (BASE_EXPONENT * norms), 0.0)
    return base + np.einsum("nm,nmk->nk", resp, cols), resp


def sb_grad_many(base, axes, cols, dirs, up):
    """appearance.py:127-163: gradients (d base, d axes, d colours, d view)."""
    ax = _effective_axes(axes)
    norms = np.linalg.norm(ax, axis=-1)
    units = ax / norms[..., None]
    w = np.clip(np.einsum("nmk,nk->nm", units, dirs), 0.0, 1.0)
    expo = BASE_EXPONENT * norms
    act = w > 1e-12
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        resp = np.where(act, w**expo, 0.0)
        resp_dw = np.where(act, expo * w ** (expo - 1.0), 0.0)
        log_w = np.where(act, np.log(np.maximum(w, 1e-300)), 0.0)
    d_resp = np.einsum("nk,nmk->nm", up, cols)
    d_cols = resp[..., None] * up[:, None, :]
    d_w = d_resp * resp_dw
    d_norm = d_resp * resp * log_w * BASE_EXPONENT
    d_units = d_w[..., None] * dirs[:, None, :]
    d_axes = (d_units - np.einsum("nmk,nmk->nm", d_units, units)[..., None] * units) / norms[..., None]
    d_axes += d_norm[..., None] * units
    d_axes = np.where(act[..., None], d_axes, 0.0)
    return up.copy(), d_axes, d_cols, np.einsum("nm,nmk->nk", d_w, units)


def is_sb(scene):
    return getattr(scene, "sh", None) is None


def shape_to_exponent(b):
    return BASE_EXPONENT * np.exp(np.clip(b, -SHAPE_CLAMP, SHAPE_CLAMP))


# ----------------------------------------------------------------------------- binning
def depth_order(depths):
    return np.argsort(depths, kind="stable")


def tile_bins(bounds, height, width, tile=TILE):
    """Depth-ordered per-tile lists (rasterizer.py:161-191)."""
    tiles_x = (width + tile - 1) // tile
    n_tiles = tiles_x * ((height + tile - 1) // tile)
    if bounds.shape[0] == 0:
        return np.zeros(n_tiles + 1, np.int64), np.zeros(0, np.int64)
    tx0, tx1 = bounds[:, 0] // tile, bounds[:, 1] // tile
    ty0, ty1 = bounds[:, 2] // tile, bounds[:, 3] // tile
    sx = (tx1 - tx0 + 1).astype(np.int64)
    sy = (ty1 - ty0 + 1).astype(np.int64)
    counts = sx * sy
    total = int(counts.sum())
    ids = np.repeat(np.arange(bounds.shape[0], dtype=np.int64), counts)
    start = np.concatenate([[0], np.cumsum(counts)[:-1]])
    local = np.arange(total, dtype=np.int64) - np.repeat(start, counts)
    rsx = np.repeat(sx, counts)
    tile_ids = (np.repeat(ty0, counts) + local // rsx) * tiles_x + (np.repeat(tx0, counts) + local % rsx)
    lists = ids[np.argsort(tile_ids, kind="stable")]
    offsets = np.zeros(n_tiles + 1, np.int64)
    np.cumsum(np.bincount(tile_ids, minlength=n_tiles), out=offsets[1:])
    return offsets, lists


# ----------------------------------------------------------------------------- forward
def view_setup(scene, cam):
    """rasterizer.py:88-116 with the SH adapter replacing sb_eval_many."""
    pos = np.asarray(scene.positions, np.float64)
    scales = np.exp(np.asarray(scene.log_scales, np.float64))
    batch = project(pos, scene.rotations, scales, cam)
    v = batch["indices"].size
    if v == 0:
        return batch, None, None
    idx = batch["indices"]
    order = depth_order(batch["depths"])
    dirs = pos[idx] - cam.center
    dirs = dirs / np.linalg.norm(dirs, axis=-1, keepdims=True)
    if is_sb(scene):
        colors, _ = sb_eval_many(np.asarray(scene.base_colors, np.float64)[idx],
                                 np.asarray(scene.lobe_axes, np.float64)[idx],
                                 np.asarray(scene.lobe_colors, np.float64)[idx], dirs)
        basis, deg = None, None
    else:
        sh = np.asarray(scene.sh, np.float64)
        deg = int(round(np.sqrt(sh.shape[1]))) - 1
        basis = sh_basis(deg, dirs)
        colors = np.einsum("vk,vkc->vc", basis, sh[idx])
    betas = shape_to_exponent(np.asarray(scene.shapes, np.float64)[idx])
    opac = sigmoid(np.asarray(scene.opacity_raw, np.float64))[idx]
    s = dict(
        means=np.ascontiguousarray(batch["means2d"][order]),
        conics=np.ascontiguousarray(batch["conics"][order]),
        opac=np.ascontiguousarray(opac[order]),
        betas=np.ascontiguousarray(betas[order]),
        colors=np.ascontiguousarray(colors[order]),
        bounds=np.ascontiguousarray(batch["bounds"][order]),
        depths=np.ascontiguousarray(batch["depths"][order]),
    )
    return batch, order, dict(sorted=s, dirs=dirs, colors=colors, betas=betas, opac=opac, basis=basis,
                              degree=deg)


def raster_forward(s, height, width, bg, offsets, lists, core="c", threads=None, want_depth=True):
    """Dispatch one tiled forward over sorted inputs ``s`` (dict from view_setup)."""
    threads = threads or (os.cpu_count() or 1)
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    v = s["means"].shape[0]
    if core == "ref":
        raw, alpha, trans, contrib = ref_core().forward_tiled(
            s["means"], s["conics"], s["opac"], s["betas"], s["colors"], s["bounds"], height, width,
            bg, TILE, offsets, lists, threads, ALPHA_MIN, T_STOP)
        return dict(raw=raw, alpha=alpha, T=trans, contrib=contrib)
    lib = c_core()
    raw = np.zeros((height, width, 3))
    trans = np.ones((height, width))
    depth = np.zeros((height, width)) if want_depth else None
    contrib = np.zeros(v, np.int64)
    count = np.zeros((height, width), np.int32)
    last = np.full((height, width), -1, np.int64)
    pairs = np.zeros((height, width), np.int64)
    lib.oracle_forward_tiled(
        v, _ptr(s["means"]), _ptr(s["conics"]), _ptr(s["opac"]), _ptr(s["betas"]), _ptr(s["colors"]),
        _ptr(s["depths"]) if want_depth else None, _ptr(s["bounds"]), height, width, _ptr(bg), TILE,
        _ptr(offsets), _ptr(lists), int(lists.size), threads, ALPHA_MIN, T_STOP,
        _ptr(raw), _ptr(trans), _ptr(depth), _ptr(contrib), _ptr(count), _ptr(last), _ptr(pairs))
    return dict(raw=raw, alpha=1.0 - trans, T=trans, depth=depth, contrib=contrib, pix_count=count,
                pix_last=last, pix_pairs=pairs)


def forward(scene, cam, bg, core="c", threads=None):
    """render_tiled (rasterizer.py:194-211) + SH colour + depth; returns a dict of fp64 arrays.

    ``contributions`` is scattered back to the full N like ``_finish`` (:132-141).
    """
    n = len(scene.positions)
    h, w = cam.height, cam.width
    bg = np.asarray(bg, np.float64)
    batch, order, shaded = view_setup(scene, cam)
    if order is None:
        raw = np.tile(bg, (h, w, 1))
        return dict(color=np.maximum(raw, 0.0), raw=raw, alpha=np.zeros((h, w)), T=np.ones((h, w)),
                    depth=np.zeros((h, w)), contributions=np.zeros(n, np.int64),
                    pix_count=np.zeros((h, w), np.int32), V=0, E=0, batch=batch, order=None,
                    offsets=np.zeros(((h + 15) // 16) * ((w + 15) // 16) + 1, np.int64),
                    lists=np.zeros(0, np.int64))
    s = shaded["sorted"]
    offsets, lists = tile_bins(s["bounds"], h, w)
    out = raster_forward(s, h, w, bg, offsets, lists, core=core, threads=threads)
    contributions = np.zeros(n, np.int64)
    contributions[batch["indices"][order]] = out["contrib"]
    out.update(color=np.maximum(out["raw"], 0.0), contributions=contributions, V=int(order.size),
               E=int(lists.size), batch=batch, order=order, offsets=offsets, lists=lists,
               shaded=shaded)
    return out


# ----------------------------------------------------------------------------- backward
def rotation_grad_to_quat(quats, g_rot):
    nrm = np.linalg.norm(quats, axis=-1, keepdims=True)
    qh = quats / nrm
    w, x, y, z = qh[:, 0], qh[:, 1], qh[:, 2], qh[:, 3]
    # dR/dq_hat contracted with g_rot, written out per component
    g = g_rot
    gw = 2.0 * (-z * g[:, 0, 1] + y * g[:, 0, 2] + z * g[:, 1, 0] - x * g[:, 1, 2] - y * g[:, 2, 0]
                + x * g[:, 2, 1])
    gx = 2.0 * (y * g[:, 0, 1] + z * g[:, 0, 2] + y * g[:, 1, 0] - 2 * x * g[:, 1, 1] - w * g[:, 1, 2]
                + z * g[:, 2, 0] + w * g[:, 2, 1] - 2 * x * g[:, 2, 2])
    gy = 2.0 * (-2 * y * g[:, 0, 0] + x * g[:, 0, 1] + w * g[:, 0, 2] + x * g[:, 1, 0] + z * g[:, 1, 2]
                - w * g[:, 2, 0] + z * g[:, 2, 1] - 2 * y * g[:, 2, 2])
    gz = 2.0 * (-2 * z * g[:, 0, 0] - w * g[:, 0, 1] + x * g[:, 0, 2] + w * g[:, 1, 0]
                - 2 * z * g[:, 1, 1] + y * g[:, 1, 2] + x * g[:, 2, 0] + y * g[:, 2, 1])
    g_qh = np.stack([gw, gx, gy, gz], axis=-1)
    return (g_qh - np.sum(g_qh * qh, axis=-1, keepdims=True) * qh) / nrm


def project_backward(positions, rotations, scales, cam, batch, d_means2d, d_cov2d):
    idx = batch["indices"]
    quats = np.asarray(rotations, np.float64)[idx]
    s = np.asarray(scales, np.float64)[idx]
    t = batch["cam_points"]
    tx, ty, tz = t[:, 0], t[:, 1], t[:, 2]
    fx, fy = cam.fx, cam.fy
    jac = pinhole_jacobian(t, cam)
    a = jac @ cam.rotation
    rot = quat_to_rotation(quats)
    sigma = (rot * (s**2)[:, None, :]) @ np.swapaxes(rot, -1, -2)
    g_m = 0.5 * (d_cov2d + np.swapaxes(d_cov2d, -1, -2))
    g_sigma = np.swapaxes(a, -1, -2) @ g_m @ a
    g_jac = (2.0 * g_m @ a @ sigma) @ cam.rotation.T
    g_t = np.einsum("vij,vi->vj", jac, d_means2d)
    g_t[:, 0] += g_jac[:, 0, 2] * (-fx / tz**2)
    g_t[:, 1] += g_jac[:, 1, 2] * (-fy / tz**2)
    g_t[:, 2] += (g_jac[:, 0, 0] * (-fx / tz**2) + g_jac[:, 0, 2] * (2.0 * fx * tx / tz**3)
                  + g_jac[:, 1, 1] * (-fy / tz**2) + g_jac[:, 1, 2] * (2.0 * fy * ty / tz**3))
    d_pos = g_t @ cam.rotation
    g_rot = 2.0 * g_sigma @ (rot * (s**2)[:, None, :])
    g_d = np.einsum("vji,vjk,vki->vi", rot, g_sigma, rot)
    return d_pos, rotation_grad_to_quat(quats, g_rot), g_d * 2.0 * s**2


def raster_backward(s, height, width, bg, raw, d_raw, offsets, lists, core="c", threads=None,
                    raw_depth=None, d_depth=None):
    threads = threads or (os.cpu_count() or 1)
    bg = np.ascontiguousarray(bg, np.float64)
    raw = np.ascontiguousarray(raw, np.float64)
    d_raw = np.ascontiguousarray(d_raw, np.float64)
    v = s["means"].shape[0]
    if core == "ref":
        dm, dc, do, db, dcol = ref_core().backward(
            s["means"], s["conics"], s["opac"], s["betas"], s["colors"], s["bounds"], height, width,
            bg, raw, d_raw, TILE, offsets, lists, threads, ALPHA_MIN, T_STOP)
        return dm, dc, do, db, dcol, np.zeros(v)
    lib = c_core()
    dm, dc, do, db, dcol, dz = (np.zeros((v, 2)), np.zeros((v, 3)), np.zeros(v), np.zeros(v),
                               np.zeros((v, 3)), np.zeros(v))
    if d_depth is not None:
        d_depth = np.ascontiguousarray(d_depth, np.float64)
        raw_depth = np.ascontiguousarray(raw_depth, np.float64)
    lib.oracle_backward(
        v, _ptr(s["means"]), _ptr(s["conics"]), _ptr(s["opac"]), _ptr(s["betas"]), _ptr(s["colors"]),
        _ptr(s["depths"]), _ptr(s["bounds"]), height, width, _ptr(bg), _ptr(raw), _ptr(raw_depth),
        _ptr(d_raw), _ptr(d_depth), TILE, _ptr(offsets), _ptr(lists), int(lists.size), threads,
        ALPHA_MIN, T_STOP, _ptr(dm), _ptr(dc), _ptr(do), _ptr(db), _ptr(dcol), _ptr(dz))
    return dm, dc, do, db, dcol, dz


def backward(scene, cam, bg, d_color, fwd, core="c", threads=None, d_depth=None):
    """render_backward (rasterizer.py:230-321) with the SH colour chain and depth.

    Returns a dict of per-parameter gradients aligned with the full N (zeros for culled),
    plus ``screen_grad_norm``.
    """
    n = len(scene.positions)
    pos = np.asarray(scene.positions, np.float64)
    grads = dict(positions=np.zeros((n, 3)), rotations=np.zeros((n, 4)), log_scales=np.zeros((n, 3)),
                 opacity_raw=np.zeros(n), shapes=np.zeros(n), screen_grad_norm=np.zeros(n))
    if is_sb(scene):
        m = scene.lobe_axes.shape[1]
        grads.update(base_colors=np.zeros((n, 3)), lobe_axes=np.zeros((n, m, 3)), lobe_colors=np.zeros((n, m, 3)))
    else:
        grads["sh"] = np.zeros((n, scene.sh.shape[1], 3))
    order = fwd["order"]
    if order is None:
        return grads
    batch, shaded = fwd["batch"], fwd["shaded"]
    s = shaded["sorted"]
    h, w = cam.height, cam.width
    d_raw = np.where(fwd["raw"] >= 0.0, d_color, 0.0)
    dm_s, dc_s, do_s, db_s, dcol_s, dz_s = raster_backward(
        s, h, w, bg, fwd["raw"], d_raw, fwd["offsets"], fwd["lists"], core=core, threads=threads,
        raw_depth=fwd.get("depth"), d_depth=d_depth)
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    d_means2d, d_conics, d_opac, d_betas, d_colors, d_z = (
        dm_s[inv], dc_s[inv], do_s[inv], db_s[inv], dcol_s[inv], dz_s[inv])
    idx = batch["indices"]
    grads["screen_grad_norm"][idx] = np.linalg.norm(d_means2d, axis=-1)
    dirs = shaded["dirs"]
    if is_sb(scene):  # rasterizer.py:275-284
        d_base, d_axes, d_cols, d_view = sb_grad_many(
            np.asarray(scene.base_colors, np.float64)[idx], np.asarray(scene.lobe_axes, np.float64)[idx],
            np.asarray(scene.lobe_colors, np.float64)[idx], dirs, d_colors)
        grads["base_colors"][idx] = d_base
        grads["lobe_axes"][idx] = d_axes
        grads["lobe_colors"][idx] = d_cols
    else:
        # SH chain: d_sh = basis (x) d_rgb ; d_dir = dbasis^T (sh . d_rgb)   (appearance.py:310-318)
        grads["sh"][idx] = shaded["basis"][:, :, None] * d_colors[:, None, :]
        sh = np.asarray(scene.sh, np.float64)[idx]
        d_basis = np.einsum("vkc,vc->vk", sh, d_colors)
        d_view = np.einsum("vkj,vk->vj", sh_basis_grad(shaded["degree"], dirs), d_basis)
    delta = pos[idx] - cam.center
    nrm = np.linalg.norm(delta, axis=-1, keepdims=True)
    d_pos_view = (d_view - np.einsum("vk,vk->v", d_view, dirs)[:, None] * dirs) / nrm
    o = shaded["opac"]
    grads["opacity_raw"][idx] = d_opac * o * (1.0 - o)
    b = np.asarray(scene.shapes, np.float64)[idx]
    d_shape = d_betas * shaded["betas"]
    d_shape[np.abs(b) > SHAPE_CLAMP] = 0.0
    grads["shapes"][idx] = d_shape
    cn = batch["conics"]
    g = np.empty((idx.size, 2, 2))
    g[:, 0, 0], g[:, 0, 1], g[:, 1, 0], g[:, 1, 1] = d_conics[:, 0], d_conics[:, 1] / 2.0, \
        d_conics[:, 1] / 2.0, d_conics[:, 2]
    inv_cov = np.empty_like(g)
    inv_cov[:, 0, 0], inv_cov[:, 0, 1], inv_cov[:, 1, 0], inv_cov[:, 1, 1] = cn[:, 0], cn[:, 1], \
        cn[:, 1], cn[:, 2]
    d_cov2d = -inv_cov @ g @ inv_cov
    scales = np.exp(np.asarray(scene.log_scales, np.float64))
    d_pos, d_rot, d_logs = project_backward(pos, scene.rotations, scales, cam, batch, d_means2d, d_cov2d)
    # depth = camera-space z = R[2] . p + t[2]  ->  d p += d_z * R[2]
    d_pos = d_pos + d_z[:, None] * cam.rotation[2][None, :]
    grads["positions"][idx] = d_pos + d_pos_view
    grads["rotations"][idx] = d_rot
    grads["log_scales"][idx] = d_logs
    return grads


# ----------------------------------------------------------------------------- loss / Adam
def gaussian_window(size=11, sigma=1.5):
    x = np.arange(size) - (size - 1) / 2.0
    w = np.exp(-(x**2) / (2.0 * sigma**2))
    return w / w.sum()


def blur(img):
    from scipy.ndimage import correlate1d

    win = gaussian_window()
    return correlate1d(correlate1d(img, win, axis=0, mode="constant"), win, axis=1, mode="constant")


SSIM_C1 = 0.01**2
SSIM_C2 = 0.03**2


def ssim(a, b):
    """training.py:51-83: mean SSIM and d/d a."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    mu_a, mu_b = blur(a), blur(b)
    qa, qab = blur(a * a), blur(a * b)
    var_b = blur(b * b) - mu_b**2
    a1 = 2.0 * mu_a * mu_b + SSIM_C1
    a2 = 2.0 * (qab - mu_a * mu_b) + SSIM_C2
    b1 = mu_a**2 + mu_b**2 + SSIM_C1
    b2 = (qa - mu_a**2) + var_b + SSIM_C2
    s = (a1 * a2) / (b1 * b2)
    d_mu = (2.0 * mu_b * (a2 - a1)) / (b1 * b2) - s * (2.0 * mu_a / b1 - 2.0 * mu_a / b2)
    d_qa = -s / b2
    d_qab = 2.0 * a1 / (b1 * b2)
    grad = (blur(d_mu) + 2.0 * a * blur(d_qa) + b * blur(d_qab)) / s.size
    return float(s.mean()), grad


def loss(rendered, target, lambda_ssim=0.2):
    """training.py:98-131 with lambda_opacity = lambda_scale = 0: (value, d_image)."""
    diff = rendered - target
    l1 = float(np.mean(np.abs(diff)))
    sv, sg = ssim(rendered, target)
    value = (1.0 - lambda_ssim) * l1 + lambda_ssim * (1.0 - sv)
    d_image = (1.0 - lambda_ssim) * np.sign(diff) / diff.size - lambda_ssim * sg
    return value, d_image


ADAM_B1, ADAM_B2, ADAM_EPS = 0.9, 0.999, 1e-15


def adam_step(params: dict, grads: dict, m: dict, v: dict, step: int, lrs: dict):
    """training.py:258-273, in place; ``step`` is the post-increment step count."""
    c1 = 1.0 - ADAM_B1**step
    c2 = 1.0 - ADAM_B2**step
    for name, p in params.items():
        g = grads[name]
        m[name] *= ADAM_B1
        m[name] += (1.0 - ADAM_B1) * g
        v[name] *= ADAM_B2
        v[name] += (1.0 - ADAM_B2) * g * g
        p -= lrs[name] * (m[name] / c1) / (np.sqrt(v[name] / c2) + ADAM_EPS)
