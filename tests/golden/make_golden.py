"""Generate golden vectors by running the REFERENCE package itself (this container only).

    python tests/golden/make_golden.py            # needs /root/reference and `make -C oracle ref`

The reference ``betasplat`` package is imported from /root/reference/pkg/src with its
compiled raster core (built from its own _raster.pyx by oracle/Makefile into oracle/_ref/)
injected as ``betasplat._raster``.  The reference's render path shades with Spherical-Beta
colour; SURVEY.md section 8(c) prescribes a small SH adapter that composes reference
functions only (project_arrays, _depth_order, sh_basis, _sh_basis_grad,
shape_to_exponent, tile_bins, core.forward_tiled / core.backward, project_backward,
training.loss / ssim / adam_step) -- it is written below, line for line after
rasterizer.py:88-321 with the two colour changes.

Outputs (small, committed): tests/golden/*.npz.  The GPU box never runs this script.
"""

from __future__ import annotations

import importlib.util
import glob
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(REPO, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    hits = glob.glob(os.path.join(REPO, "oracle", "_ref", "_raster*.so"))
    if not hits:
        raise SystemExit("build the reference core first: make -C oracle ref")
    sys.path.insert(0, REF_SRC)
    spec = importlib.util.spec_from_file_location("betasplat._raster", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    sys.modules["betasplat._raster"] = mod
    import betasplat  # noqa: F401
    from betasplat import backend

    assert backend.HAVE_COMPILED and backend.get_core().COMPILED
    return betasplat


def ref_primitives(bs, scene):
    """PrimitiveSet with M = 0 lobes; SH coefficients are carried separately."""
    from betasplat.primitive import PrimitiveSet

    n = len(scene.positions)
    return PrimitiveSet(
        positions=scene.positions.astype(np.float64),
        opacity_raw=scene.opacity_raw.astype(np.float64),
        rotations=scene.rotations.astype(np.float64),
        log_scales=scene.log_scales.astype(np.float64),
        shapes=scene.shapes.astype(np.float64),
        base_colors=np.zeros((n, 3)),
        lobe_axes=np.zeros((n, 0, 3)),
        lobe_colors=np.zeros((n, 0, 3)),
    )


def ref_camera(cam):
    from betasplat.primitive import Camera

    return Camera(cam.world_to_camera.copy(), cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)


def sh_view_setup(prims, sh, camera):
    """rasterizer.py:88-103 with colour = einsum(sh_basis(deg, dirs), sh[idx])."""
    from betasplat.appearance import sh_basis
    from betasplat.kernel import shape_to_exponent
    from betasplat.primitive import project_arrays
    from betasplat.rasterizer import _depth_order

    batch = project_arrays(prims.positions, prims.rotations, prims.scales, camera)
    if batch.count == 0:
        return batch, None, None, None
    order = _depth_order(batch.depths)
    view_dirs = prims.positions[batch.indices] - camera.center
    view_dirs = view_dirs / np.linalg.norm(view_dirs, axis=-1, keepdims=True)
    deg = int(round(np.sqrt(sh.shape[1]))) - 1
    colors = np.einsum("vk,vkc->vc", sh_basis(deg, view_dirs), sh[batch.indices])
    betas = shape_to_exponent(prims.shapes[batch.indices])
    return batch, order, view_dirs, (colors, betas)


def sh_render_tiled(prims, sh, camera, bg, threads=8):
    """rasterizer.py:194-211 through the SH view setup; also returns the binning."""
    from betasplat import backend
    from betasplat.rasterizer import ALPHA_MIN, T_STOP, TILE_SIZE, _finish, _sorted_inputs, tile_bins

    core = backend.get_core()
    batch, order, _, shaded = sh_view_setup(prims, sh, camera)
    means, conics, opac, betas, colors, bounds = _sorted_inputs(prims, batch, order, shaded)
    offsets, lists = tile_bins(bounds, camera.height, camera.width)
    raw, alpha, trans, contrib = core.forward_tiled(
        means, conics, opac, betas, colors, bounds, camera.height, camera.width, bg, TILE_SIZE,
        offsets, lists, threads, ALPHA_MIN, T_STOP)
    out = _finish(prims, batch, order, raw, alpha, trans, contrib)
    return out, dict(indices=batch.indices, order=order, bounds=bounds, depths=batch.depths[order],
                     means=means, conics=conics, opac=opac, betas=betas, colors=colors,
                     offsets=offsets, lists=lists)


def sh_render_backward(prims, sh, camera, bg, d_color, fwd, threads=8):
    """rasterizer.py:230-321 with the SH colour chain (appearance.py:264-318)."""
    from betasplat import backend
    from betasplat.appearance import _sh_basis_grad, sh_basis
    from betasplat.kernel import SHAPE_CLAMP
    from betasplat.primitive import project_backward
    from betasplat.rasterizer import ALPHA_MIN, T_STOP, TILE_SIZE, _sorted_inputs, tile_bins

    core = backend.get_core()
    n = len(prims)
    grads = {k: np.zeros_like(v) for k, v in prims.parameters().items()}
    grads["sh"] = np.zeros_like(sh)
    batch, order, view_dirs, shaded = sh_view_setup(prims, sh, camera)
    means, conics, opac, betas, colors, bounds = _sorted_inputs(prims, batch, order, shaded)
    offsets, lists = tile_bins(bounds, camera.height, camera.width)
    d_raw = np.ascontiguousarray(np.where(fwd.raw_color >= 0.0, d_color, 0.0), dtype=np.float64)
    dm, dc, do, db, dcol = core.backward(
        means, conics, opac, betas, colors, bounds, camera.height, camera.width, bg,
        np.ascontiguousarray(fwd.raw_color), d_raw, TILE_SIZE, offsets, lists, threads, ALPHA_MIN, T_STOP)
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    d_means2d, d_conics, d_opac, d_betas, d_colors = dm[inv], dc[inv], do[inv], db[inv], dcol[inv]
    idx = batch.indices
    deg = int(round(np.sqrt(sh.shape[1]))) - 1
    basis = sh_basis(deg, view_dirs)
    grads["sh"][idx] = basis[:, :, None] * d_colors[:, None, :]
    d_basis = np.einsum("vkc,vc->vk", sh[idx], d_colors)
    d_view = np.einsum("vkj,vk->vj", _sh_basis_grad(deg, view_dirs), d_basis)
    delta = prims.positions[idx] - camera.center
    norm = np.linalg.norm(delta, axis=-1, keepdims=True)
    d_pos_view = (d_view - np.einsum("vk,vk->v", d_view, view_dirs)[:, None] * view_dirs) / norm
    o = opac[inv]
    grads["opacity_raw"][idx] = d_opac * o * (1.0 - o)
    d_shape = d_betas * shaded[1]
    d_shape[np.abs(prims.shapes[idx]) > SHAPE_CLAMP] = 0.0
    grads["shapes"][idx] = d_shape
    g_inv = np.empty((batch.count, 2, 2))
    g_inv[:, 0, 0] = d_conics[:, 0]
    g_inv[:, 0, 1] = d_conics[:, 1] / 2.0
    g_inv[:, 1, 0] = d_conics[:, 1] / 2.0
    g_inv[:, 1, 1] = d_conics[:, 2]
    inv_cov = np.empty_like(g_inv)
    inv_cov[:, 0, 0] = batch.conics[:, 0]
    inv_cov[:, 0, 1] = batch.conics[:, 1]
    inv_cov[:, 1, 0] = batch.conics[:, 1]
    inv_cov[:, 1, 1] = batch.conics[:, 2]
    d_cov2d = -inv_cov @ g_inv @ inv_cov
    d_pos, d_rot, d_logs = project_backward(prims.positions, prims.rotations, prims.scales, camera,
                                            batch, d_means2d, d_cov2d)
    grads["positions"][idx] = d_pos + d_pos_view
    grads["rotations"][idx] = d_rot
    grads["log_scales"][idx] = d_logs
    del n
    return grads


def main():
    bs = import_reference()
    sys.path.insert(0, REPO)
    from paper_2501_18630_b200.scenes import make_workload, SplatScene
    from betasplat import training

    os.makedirs(OUT, exist_ok=True)
    white = np.ones(3)

    # ---- G1: config 0 forward at full size (N=10k, SH0, 256^2)
    wl = make_workload("c0", seed=0)
    cam = wl.cameras[0]
    prims = ref_primitives(bs, wl.scene)
    sh = wl.scene.sh.astype(np.float64)
    out, bins = sh_render_tiled(prims, sh, ref_camera(cam), white)
    np.savez_compressed(
        os.path.join(OUT, "c0_forward.npz"),
        **wl.scene.arrays(), w2c=cam.world_to_camera, intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
        size=np.array([cam.width, cam.height]), bg=white,
        raw=out.raw_color, T=out.transmittance, contributions=out.contributions,
        indices=bins["indices"], order=bins["order"], bounds=bins["bounds"], depths=bins["depths"],
        offsets=bins["offsets"], lists=bins["lists"], colors=bins["colors"])

    # ---- G2: small SH-3 scene (config-1 distribution), forward + backward under N(0,1) upstream
    wl = make_workload("c1", seed=3, n=3000, width=96, height=80)
    cam = wl.cameras[0]
    prims = ref_primitives(bs, wl.scene)
    sh = wl.scene.sh.astype(np.float64)
    rng = np.random.default_rng(5)
    upstream = rng.standard_normal((cam.height, cam.width, 3))
    out, bins = sh_render_tiled(prims, sh, ref_camera(cam), white)
    grads = sh_render_backward(prims, sh, ref_camera(cam), white, upstream, out)
    np.savez_compressed(
        os.path.join(OUT, "sh3_fwd_bwd.npz"),
        **wl.scene.arrays(), w2c=cam.world_to_camera, intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
        size=np.array([cam.width, cam.height]), bg=white, upstream=upstream,
        raw=out.raw_color, T=out.transmittance, contributions=out.contributions,
        offsets=bins["offsets"], lists=bins["lists"], bounds=bins["bounds"],
        **{"g_" + k: v for k, v in grads.items()})

    # ---- G3: non-Gaussian shapes (b != 0), SH-2, off-centre camera, non-tile-multiple image
    rng = np.random.default_rng(11)
    n = 400
    q = rng.standard_normal((n, 4))
    scene = SplatScene(
        positions=rng.uniform(-0.8, 0.8, (n, 3)).astype(np.float32),
        rotations=(q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32),
        log_scales=np.log(rng.uniform(0.05, 0.35, (n, 3))).astype(np.float32),
        opacity_raw=rng.normal(0.0, 1.5, n).astype(np.float32),
        shapes=rng.uniform(-1.5, 1.5, n).astype(np.float32),
        sh=rng.normal(0.0, 0.4, (n, 9, 3)).astype(np.float32))
    from paper_2501_18630_b200.camera import Camera

    cam = Camera.from_lookat((0.3, 0.5, -4.0), (0, 0, 0), (0, 1, 0), 0.9, 70, 50)
    prims = ref_primitives(bs, scene)
    sh = scene.sh.astype(np.float64)
    upstream = rng.standard_normal((cam.height, cam.width, 3))
    out, bins = sh_render_tiled(prims, sh, ref_camera(cam), white)
    grads = sh_render_backward(prims, sh, ref_camera(cam), white, upstream, out)
    np.savez_compressed(
        os.path.join(OUT, "shapes_sh2.npz"),
        **scene.arrays(), w2c=cam.world_to_camera, intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
        size=np.array([cam.width, cam.height]), bg=white, upstream=upstream,
        raw=out.raw_color, T=out.transmittance, contributions=out.contributions,
        offsets=bins["offsets"], lists=bins["lists"], bounds=bins["bounds"],
        **{"g_" + k: v for k, v in grads.items()})

    # ---- G4: loss (0.8 L1 + 0.2 D-SSIM) and its image gradient (training.py:98-131)
    rng = np.random.default_rng(7)
    a = rng.uniform(0.0, 1.0, (40, 52, 3)).astype(np.float32).astype(np.float64)
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1).astype(np.float32).astype(np.float64)

    class Cfg:
        lambda_ssim = 0.2
        lambda_opacity = 0.0
        lambda_scale = 0.0

    value, d_image, _ = training.loss(a, b, prims, Cfg())
    sval, sgrad = training.ssim(a, b)
    np.savez_compressed(os.path.join(OUT, "loss.npz"), a=a, b=b, value=value, d_image=d_image,
                        ssim=sval, ssim_grad=sgrad)

    # ---- G5: Adam (training.py:258-273), three steps on every parameter group
    from betasplat.primitive import PrimitiveSet

    rng = np.random.default_rng(9)
    n = 64
    p0 = PrimitiveSet(positions=rng.normal(size=(n, 3)), opacity_raw=rng.normal(size=n),
                      rotations=rng.normal(size=(n, 4)), log_scales=rng.normal(size=(n, 3)),
                      shapes=rng.normal(size=n), base_colors=rng.normal(size=(n, 3)),
                      lobe_axes=np.zeros((n, 0, 3)), lobe_colors=np.zeros((n, 0, 3)))
    p = p0.copy()
    state = training.AdamState.zeros_for(p)
    lrs = {k: (1.6e-4 if k == "positions" else 5e-3) for k in p.parameters()}
    gs = []
    for _ in range(3):
        g = {k: rng.normal(size=v.shape) for k, v in p.parameters().items()}
        gs.append(g)
        training.adam_step(p, g, state, lrs)
    save = {}
    for k in ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "base_colors"):
        save["p0_" + k] = getattr(p0, k)
        save["p3_" + k] = getattr(p, k)
        for i, g in enumerate(gs):
            save[f"g{i}_" + k] = g[k]
    np.savez_compressed(os.path.join(OUT, "adam.npz"), **save)
    # ---- G6: the reference's DEFAULT path (Spherical-Beta colour), unmodified render_tiled /
    #      render_backward, on its own random-scene distribution (tests/conftest.py:15-31)
    from betasplat import rasterizer as rz
    from betasplat.primitive import PrimitiveSet as RefPS
    from paper_2501_18630_b200.scenes import sb_random_scene

    for name, seed, n, (w, h), lobes in (("sb_small.npz", 21, 60, (48, 40), 2),
                                         ("sb_medium.npz", 22, 1500, (96, 72), 3)):
        rng = np.random.default_rng(seed)
        sc = sb_random_scene(rng, n, lobes=lobes)
        ref = RefPS(**{k: v.astype(np.float64) for k, v in sc.arrays().items()})
        from paper_2501_18630_b200.camera import Camera

        cam = Camera.from_lookat((0.2, -0.3, -4.0), (0, 0, 0), (0, 1, 0), 0.9, w, h)
        up = rng.standard_normal((h, w, 3))
        out = rz.render_tiled(ref, ref_camera(cam), white)
        gr = rz.render_backward(ref, ref_camera(cam), white, up, forward_out=out)
        np.savez_compressed(
            os.path.join(OUT, name), **sc.arrays(), w2c=cam.world_to_camera,
            intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]), size=np.array([cam.width, cam.height]),
            bg=white, upstream=up, color=out.color, raw=out.raw_color, T=out.transmittance,
            contributions=out.contributions, **{"g_" + k: v for k, v in gr.parameters().items()},
            g_screen_grad_norm=gr.screen_grad_norm)
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
