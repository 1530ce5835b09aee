"""GPU parity: libbsr.so (through the C-ABI) against the oracle on identical seeded inputs.

Bars (BASELINE.json north_star): tile keys / sort order / binning / contributions /
per-pixel counts BIT-EXACT; images within 1e-4 absolute (fp32); gradients within
1e-3 relative / 1e-5 absolute (atol scaled by max|g| per group like the reference's FD
test, tests/test_rasterizer.py:279-282).
"""

import numpy as np
import pytest

from conftest import golden, golden_scene_camera, random_scene, toy_camera

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4


def _gpu_prims(scene):
    from paper_2501_18630_b200 import PrimitiveSet

    if getattr(scene, "sh", None) is None:  # Spherical-Beta colour (the reference's default)
        return PrimitiveSet.from_reference(scene)
    return PrimitiveSet.from_scene(scene)


def _oracle_fwd(scene, cam, bg):
    from oracle import pipeline as orc

    return orc.forward(scene, cam, bg, core="c")


def _compare_forward(scene, cam, bg, cuda, check_bins=True):
    from paper_2501_18630_b200 import render_tiled
    from paper_2501_18630_b200.rasterizer import debug_export

    ref = _oracle_fwd(scene, cam, bg)
    out = render_tiled(_gpu_prims(scene), cam, bg)
    np.testing.assert_array_equal(out.contributions.cpu().numpy(), ref["contributions"])
    np.testing.assert_array_equal(out.pixel_count.cpu().numpy(), ref["pix_count"])
    assert np.abs(out.raw_color.cpu().numpy() - ref["raw"]).max() <= IMG_TOL
    assert np.abs(out.color.cpu().numpy() - ref["color"]).max() <= IMG_TOL
    assert np.abs(out.transmittance.cpu().numpy() - ref["T"]).max() <= IMG_TOL
    assert np.abs(out.alpha.cpu().numpy() - ref["alpha"]).max() <= IMG_TOL
    zscale = max(1.0, float(np.abs(ref["depth"]).max()))
    assert np.abs(out.depth.cpu().numpy() - ref["depth"]).max() <= IMG_TOL * zscale
    if check_bins and ref["order"] is not None:
        dbg = debug_export(out.frame)
        assert dbg["visible"] == ref["V"] and dbg["entries"] == ref["E"]
        np.testing.assert_array_equal(dbg["src"], ref["batch"]["indices"])
        np.testing.assert_array_equal(dbg["order"], ref["order"])
        np.testing.assert_array_equal(dbg["bounds"], ref["batch"]["bounds"])
        np.testing.assert_array_equal(dbg["lists"], ref["order"][ref["lists"]])
        off = ref["offsets"]
        np.testing.assert_array_equal(dbg["ranges"][:, 1] - dbg["ranges"][:, 0], np.diff(off))
        nz = np.diff(off) > 0
        np.testing.assert_array_equal(dbg["ranges"][nz, 0], off[:-1][nz])
    return out, ref


@pytest.mark.parametrize("name", ["c0_forward.npz", "sh3_fwd_bwd.npz", "shapes_sh2.npz"])
def test_forward_golden_scenes(cuda, name):
    g = golden(name)
    scene, cam = golden_scene_camera(g)
    out, ref = _compare_forward(scene, cam, g["bg"], cuda)
    # and against the reference's own golden vectors
    np.testing.assert_array_equal(out.contributions.cpu().numpy(), g["contributions"])
    assert np.abs(out.raw_color.cpu().numpy() - g["raw"]).max() <= IMG_TOL


def test_forward_config1_full_size(cuda):
    from paper_2501_18630_b200.scenes import make_workload

    wl = make_workload("c1", seed=0)
    _compare_forward(wl.scene, wl.cameras[0], wl.background, cuda)


def test_forward_config2_reduced(cuda):
    from paper_2501_18630_b200.scenes import make_workload

    wl = make_workload("c2", seed=0, n=200_000, width=960, height=540)
    _compare_forward(wl.scene, wl.cameras[0], wl.background, cuda)


@pytest.mark.parametrize("seed,n,w,h", [(14, 1, 70, 50), (15, 7, 70, 50), (16, 60, 70, 50),
                                        (17, 300, 70, 50), (18, 20, 16, 16), (19, 120, 96, 64)])
def test_forward_random_scenes(cuda, seed, n, w, h):
    """tests/test_rasterizer.py:150-166 analogues (non tile-multiple, single tile)."""
    rng = np.random.default_rng(seed)
    scene = random_scene(rng, n, degree=1 + seed % 3)
    _compare_forward(scene, toy_camera(w, h), np.ones(3), cuda)


def test_depth_ties_and_fp32_collisions(cuda):
    """Exact and fp32-colliding depths: order must equal np.argsort(fp64 depth, stable)."""
    rng = np.random.default_rng(41)
    n = 400
    scene = random_scene(rng, n, degree=0, spread=0.6)
    # groups of identical depths (index tie-break) and depths 1e-8 apart (same fp32 key)
    z = np.repeat(rng.uniform(-0.5, 0.5, n // 8), 8).astype(np.float32)
    z[: n // 2] = (np.arange(n // 2) % 37 * 1e-8).astype(np.float32)
    rng.shuffle(z)
    scene.positions[:, 2] = z
    _compare_forward(scene, toy_camera(64, 64), np.ones(3), cuda)


def test_empty_and_culled_scenes(cuda):
    from paper_2501_18630_b200 import render_tiled

    cam = toy_camera()
    rng = np.random.default_rng(3)
    scene = random_scene(rng, 10)
    scene.positions[:, 2] = -10.0  # everything behind the camera (eye at z=-4 looking +z)
    out = render_tiled(_gpu_prims(scene), cam, np.ones(3))
    np.testing.assert_array_equal(out.color.cpu().numpy(), np.ones((32, 32, 3), np.float32))
    np.testing.assert_array_equal(out.alpha.cpu().numpy(), np.zeros((32, 32), np.float32))
    assert int(out.contributions.sum()) == 0
    empty = scene.take(np.zeros(0, dtype=np.int64))
    out = render_tiled(_gpu_prims(empty), cam, np.ones(3))
    np.testing.assert_array_equal(out.color.cpu().numpy(), np.ones((32, 32, 3), np.float32))


def test_extinction_alpha_near_one(cuda):
    """tests/test_rasterizer.py:68-90: opacity 1 - 1e-12 (fp64 replay path)."""
    from paper_2501_18630_b200.scenes import SplatScene
    from paper_2501_18630_b200 import render_tiled

    cam = toy_camera(33, 33)

    def mk(zs, cols, ops):
        n = len(zs)
        sh = np.asarray(cols, np.float64)[:, None, :] / 0.28209479177387814
        op = np.asarray(ops, np.float64)
        return SplatScene(positions=np.array([[0, 0, z] for z in zs], np.float32),
                          rotations=np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)),
                          log_scales=np.log(np.full((n, 3), 0.3)).astype(np.float32),
                          opacity_raw=(np.log(op) - np.log1p(-op)).astype(np.float32),
                          shapes=np.full(n, -2.0, np.float32), sh=sh.astype(np.float32))

    front = mk([0.0], [[1, 0, 0]], [1 - 1e-12])
    both = mk([0.0, 1.0], [[1, 0, 0], [1, 1, 1]], [1 - 1e-12, 0.9])
    a = render_tiled(_gpu_prims(front), cam, np.zeros(3))
    b = render_tiled(_gpu_prims(both), cam, np.zeros(3))
    np.testing.assert_array_equal(a.color.cpu().numpy()[16, 16], b.color.cpu().numpy()[16, 16])
    for s in (front, both):
        _compare_forward(s, cam, np.zeros(3), cuda)


def test_core_seam_forward_matches_reference_core(cuda):
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import backend

    core = backend.get_core("cuda")
    g = golden("sh3_fwd_bwd.npz")
    scene, cam = golden_scene_camera(g)
    _, order, shaded = orc.view_setup(scene, cam)
    s = shaded["sorted"]
    off, lists = orc.tile_bins(s["bounds"], cam.height, cam.width)
    ref = orc.raster_forward(s, cam.height, cam.width, g["bg"], off, lists, core="c")
    raw, alpha, trans, contrib, extra = core.forward_tiled(
        s["means"], s["conics"], s["opac"], s["betas"], s["colors"], s["bounds"], cam.height, cam.width,
        g["bg"], 16, off, lists, 8, orc.ALPHA_MIN, orc.T_STOP, return_extra=True)
    np.testing.assert_array_equal(contrib, ref["contrib"])
    np.testing.assert_array_equal(extra["pixel_count"], ref["pix_count"])
    assert np.abs(raw - ref["raw"]).max() <= IMG_TOL
    assert np.abs(trans - ref["T"]).max() <= IMG_TOL
    naive = core.forward_naive(s["means"], s["conics"], s["opac"], s["betas"], s["colors"], s["bounds"],
                               cam.height, cam.width, g["bg"], orc.ALPHA_MIN, orc.T_STOP)
    np.testing.assert_array_equal(naive[3], ref["contrib"])


def _grad_close(a, b, name):
    scale = max(np.abs(b).max(), 1e-30)
    np.testing.assert_allclose(a, b, rtol=1e-3, atol=1e-5 * scale, err_msg=name)


def test_core_seam_backward_matches_reference_core(cuda):
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import backend

    core = backend.get_core("cuda")
    g = golden("shapes_sh2.npz")
    scene, cam = golden_scene_camera(g)
    _, order, shaded = orc.view_setup(scene, cam)
    s = shaded["sorted"]
    off, lists = orc.tile_bins(s["bounds"], cam.height, cam.width)
    fwd = orc.raster_forward(s, cam.height, cam.width, g["bg"], off, lists, core="c")
    d_raw = np.where(fwd["raw"] >= 0, g["upstream"], 0.0)
    ref = orc.raster_backward(s, cam.height, cam.width, g["bg"], fwd["raw"], d_raw, off, lists, core="c")
    got = core.backward(s["means"], s["conics"], s["opac"], s["betas"], s["colors"], s["bounds"],
                        cam.height, cam.width, g["bg"], fwd["raw"], d_raw, 16, off, lists, 8,
                        orc.ALPHA_MIN, orc.T_STOP)
    for name, a, b in zip(("d_means", "d_conics", "d_opac", "d_betas", "d_colors"), got, ref[:5]):
        _grad_close(a, b, name)


@pytest.mark.parametrize("name", ["sh3_fwd_bwd.npz", "shapes_sh2.npz"])
def test_backward_golden_scenes(cuda, name):
    from paper_2501_18630_b200 import render_backward, render_tiled

    g = golden(name)
    scene, cam = golden_scene_camera(g)
    prims = _gpu_prims(scene)
    out = render_tiled(prims, cam, g["bg"])
    grads = render_backward(prims, cam, g["bg"], g["upstream"].astype(np.float32), forward_out=out)
    for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"):
        _grad_close(getattr(grads, k).cpu().numpy(), g["g_" + k], k)


def test_backward_with_depth_matches_oracle(cuda):
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import render_backward, render_tiled

    rng = np.random.default_rng(31)
    scene = random_scene(rng, 150, degree=3)
    cam = toy_camera(64, 48)
    bg = np.array([0.2, 0.5, 1.0])
    up = rng.standard_normal((48, 64, 3))
    upd = rng.standard_normal((48, 64))
    fwd = orc.forward(scene, cam, bg, core="c")
    ref = orc.backward(scene, cam, bg, up, fwd, core="c", d_depth=upd)
    prims = _gpu_prims(scene)
    out = render_tiled(prims, cam, bg)
    grads = render_backward(prims, cam, bg, up.astype(np.float32), forward_out=out,
                            d_depth=upd.astype(np.float32))
    for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"):
        _grad_close(getattr(grads, k).cpu().numpy(), ref[k], k)


def _needle_scene(rng, n):
    """Long thin footprints (scale 0.8 x 0.004 x 0.004, random orientations) among ordinary
    primitives: their factored-conic bound exceeds the fp32 limit, so they take the
    compensated 'needle' evaluation (raster.cuh) or, if that bound fails too, the fp64 one."""
    scene = random_scene(rng, n, degree=2, spread=0.7, scale_range=(0.02, 0.1))
    k = n // 2
    scene.log_scales[:k] = np.log(np.array([0.8, 0.004, 0.004], np.float32))
    return scene, k


def _needle_count(scene, cam):
    """How many records the device classifies as needles (the bounds of preprocess.cu)."""
    from oracle import pipeline as orc

    b = orc.project(np.asarray(scene.positions, np.float64), scene.rotations,
                    np.exp(np.asarray(scene.log_scales, np.float64)), cam)
    c, cov = b["conics"], b["cov2d"]
    l11 = np.sqrt(c[:, 0]); l21 = c[:, 1] / l11; l22 = np.sqrt(np.maximum(c[:, 2] - l21 ** 2, 0))
    X, Y = np.sqrt(cov[:, 0, 0]) + 2, np.sqrt(cov[:, 1, 1]) + 2
    eps = 5.9604644775390625e-08
    kr = eps * 1.5 * (4 * (l11 * X + abs(l21) * Y) + 8 + 4 * l11 * X + 4 * (abs(l21) + l22) * Y)
    kn = eps * 1.5 * (12 + 8 * eps * l11 * (X + abs(l21 / l11) * Y))
    return int(np.sum((kr > 2e-5) & (kn <= 2e-5) & (l22 > 0)))


def _needle_grads(cuda):
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import render_backward, render_tiled

    rng = np.random.default_rng(97)
    scene, k = _needle_scene(rng, 240)
    cam = toy_camera(256, 192)
    bg = np.array([1.0, 1.0, 1.0])
    up = rng.standard_normal((192, 256, 3))
    fwd = orc.forward(scene, cam, bg, core="c")
    ref = orc.backward(scene, cam, bg, up, fwd, core="c")
    prims = _gpu_prims(scene)
    out = render_tiled(prims, cam, bg)
    grads = render_backward(prims, cam, bg, up.astype(np.float32), forward_out=out)
    return grads, ref, k


def test_needles_match_oracle(cuda):
    """Needle records: forward bit-exact on counts / tile lists against the oracle, images
    within tolerance; gradients of the ordinary primitives rendered together with them
    within 1e-3 (the needles' own gradients: test_needle_gradients_strict)."""
    rng = np.random.default_rng(97)
    scene, _ = _needle_scene(rng, 240)
    cam = toy_camera(256, 192)
    assert _needle_count(scene, cam) >= 20
    _compare_forward(scene, cam, np.ones(3), cuda)
    grads, ref, k = _needle_grads(cuda)
    for name in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"):
        _grad_close(getattr(grads, name).cpu().numpy()[k:], ref[name][k:], name)


def test_needle_gradients_strict(cuda):
    """The needles' own gradients within 1e-3 (their geometry partials are summed in fp64
    and their chain runs in fp64: DESIGN.md section 3, 'Gradients')."""
    grads, ref, k = _needle_grads(cuda)
    for name in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"):
        _grad_close(getattr(grads, name).cpu().numpy()[:k], ref[name][:k], name)


def test_zero_upstream_gives_zero_gradients(cuda):
    """tests/test_rasterizer.py:221-227."""
    from paper_2501_18630_b200 import render_backward

    rng = np.random.default_rng(20)
    prims = _gpu_prims(random_scene(rng, 8))
    cam = toy_camera()
    grads = render_backward(prims, cam, np.ones(3), np.zeros((32, 32, 3), np.float32))
    assert float(grads.flat.abs().max()) == 0.0


def test_occluded_primitive_gets_zero_opacity_gradient(cuda):
    """tests/test_rasterizer.py:229-252."""
    from paper_2501_18630_b200.scenes import SplatScene
    from paper_2501_18630_b200 import render_backward

    cam = toy_camera(17, 17)
    op = np.array([1 - 1e-12, 0.5])
    scene = SplatScene(positions=np.array([[0, 0, 0], [0, 0, 1.0]], np.float32),
                       rotations=np.tile(np.array([1, 0, 0, 0], np.float32), (2, 1)),
                       log_scales=np.log(np.array([[3.0] * 3, [0.05] * 3])).astype(np.float32),
                       opacity_raw=(np.log(op) - np.log1p(-op)).astype(np.float32),
                       shapes=np.full(2, -2.0, np.float32),
                       sh=np.full((2, 1, 3), 0.5 / 0.28209479177387814, np.float32))
    grads = render_backward(_gpu_prims(scene), cam, np.zeros(3), np.ones((17, 17, 3), np.float32))
    assert float(grads.opacity_raw[1]) == 0.0


def test_loss_matches_reference_golden(cuda):
    from paper_2501_18630_b200 import training

    g = golden("loss.npz")
    value, d_image = training.loss(g["a"], g["b"])
    assert value == pytest.approx(float(g["value"]), rel=1e-5)
    d = d_image.cpu().numpy()
    scale = np.abs(g["d_image"]).max()
    np.testing.assert_allclose(d, g["d_image"], rtol=1e-3, atol=1e-4 * scale)


@pytest.mark.parametrize("w,h", [(1280, 720), (2304, 1856)])
def test_loss_both_tilings_match_oracle(cuda, w, h):
    """Both SSIM tilings (one channel per CTA up to 4 Mpixel, all three above) against the
    oracle's fp64 loss (training.py:51-131) on random images."""
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import training

    rng = np.random.default_rng(w)
    a = rng.uniform(0.0, 1.0, (h, w, 3)).astype(np.float32)
    b = np.clip(a + rng.normal(0.0, 0.1, a.shape), 0.0, 1.0).astype(np.float32)
    value, d_image = training.loss(a, b)
    ref_value, ref_d = orc.loss(a.astype(np.float64), b.astype(np.float64))
    assert value == pytest.approx(ref_value, rel=1e-5)
    scale = np.abs(ref_d).max()
    np.testing.assert_allclose(d_image.cpu().numpy(), ref_d, rtol=1e-3, atol=1e-4 * scale)


def test_adam_matches_reference_golden(cuda):
    import torch
    from paper_2501_18630_b200 import training
    from paper_2501_18630_b200.primitive import GradientBuffer, PrimitiveSet

    g = golden("adam.npz")
    n = g["p0_positions"].shape[0]
    sh = np.zeros((n, 1, 3), np.float32)
    prims = PrimitiveSet(g["p0_positions"], g["p0_rotations"], g["p0_log_scales"], g["p0_opacity_raw"],
                         g["p0_shapes"], sh)
    p64 = {k: g["p0_" + k].copy() for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes")}
    state = training.AdamState(prims)
    lrs = training.group_lrs(lr_shapes=5e-3)  # the reference optimises every group
    for i in range(3):
        gb = GradientBuffer.zeros_for(prims)
        for k in p64:
            getattr(gb, k).copy_(torch.from_numpy(g[f"g{i}_" + k].astype(np.float32)))
        training.adam_step(prims, gb, state, lrs)
    for k in p64:
        np.testing.assert_allclose(getattr(prims, k).cpu().numpy(), g["p3_" + k], rtol=0, atol=2e-6, err_msg=k)


def test_train_step_graph_replay_matches_eager(cuda):
    """TrainStep (fwd + L1/D-SSIM + bwd + Adam) captured in a CUDA graph == eager steps,
    and the loss decreases (config-1 distribution, reduced size)."""
    import torch
    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.scenes import make_workload, target_scene
    from paper_2501_18630_b200.training import TrainStep, render_targets

    wl = make_workload("c1", seed=0, n=20_000, width=256, height=256)
    cams = wl.cameras
    tgt = render_targets(PrimitiveSet.from_scene(target_scene("c1", 1, 20_000)), cams, wl.background)
    a = PrimitiveSet.from_scene(wl.scene)
    b = PrimitiveSet.from_scene(wl.scene)
    sa = TrainStep(a, cams, tgt, wl.background)
    sb = TrainStep(b, cams, tgt, wl.background)
    sa.step(check=True)
    sb.step(check=True)
    la = [float(sa.loss_values[0, 0])]
    lb = [float(sb.loss_values[0, 0])]
    sb.capture(warmup=0)  # capture records (does not run) the step
    for _ in range(6):
        la.append(float(sa.step()[0, 0]))
        lb.append(float(sb.replay()[0, 0]))
    torch.cuda.synchronize()
    sa.check_frames()
    sb.check_frames()
    assert la[-1] < la[0]
    np.testing.assert_allclose(lb, la, rtol=1e-4)
    # same math, different float-atomic order: parameters agree to fp32 noise except where
    # Adam normalises a gradient that is itself at noise level
    d = np.abs(b.flat.cpu().numpy() - a.flat.cpu().numpy())
    assert np.mean(d > 1e-4) < 1e-3 and d.max() < 7 * 5e-3
    assert int(sb.adam.step_dev.item()) == 7


@pytest.mark.parametrize("name", ["sb_small.npz", "sb_medium.npz"])
def test_spherical_beta_drop_in_matches_reference(cuda, name):
    """Spherical-Beta colour: the GPU path against the UNMODIFIED reference render_tiled /
    render_backward (golden vectors from the reference package) and against the oracle."""
    from paper_2501_18630_b200 import render_backward

    g = golden(name)
    scene, cam = golden_scene_camera(g)
    out, ref = _compare_forward(scene, cam, g["bg"], cuda)
    np.testing.assert_array_equal(out.contributions.cpu().numpy(), g["contributions"])
    assert np.abs(out.color.cpu().numpy() - g["color"]).max() <= IMG_TOL
    grads = render_backward(_gpu_prims(scene), cam, g["bg"], g["upstream"].astype(np.float32))
    for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "base_colors", "lobe_axes",
              "lobe_colors"):
        _grad_close(getattr(grads, k).cpu().numpy(), g["g_" + k], k)


def test_spherical_beta_training_step(cuda):
    """TrainStep on a Spherical-Beta set with the reference's default learning rates."""
    import torch
    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.scenes import sb_random_scene
    from paper_2501_18630_b200.training import TrainStep, render_targets

    rng = np.random.default_rng(5)
    cam = toy_camera(64, 64)
    tgt = render_targets(PrimitiveSet.from_reference(sb_random_scene(rng, 200)), [cam], np.ones(3))
    prims = PrimitiveSet.from_reference(sb_random_scene(rng, 200))
    st = TrainStep(prims, [cam], tgt, np.ones(3))
    st.step(check=True)
    l0 = float(st.loss_values[0, 0])
    for _ in range(20):
        st.step()
    torch.cuda.synchronize()
    assert float(st.loss_values[0, 0]) < l0


@pytest.mark.parametrize("n,bunched", [(2500, False), (2500, True), (6000, False), (6000, True), (20000, False),
                                       (30000, False)])
def test_crowded_tile_binning(cuda, n, bunched):
    """Crowded tiles: 1024 < n <= 4096 entries take the equi-depth bucket sort in shared
    memory (also with depths bunched in a sliver of the tile's range plus far outliers),
    4096 < n <= 20480 the same sort in 160 KB of dynamic shared memory (tile_sort_big_kernel),
    beyond that the in-place network in global memory; lists, offsets and depth order stay
    bit-exact."""
    rng = np.random.default_rng(50 + n + bunched)
    scene = random_scene(rng, n, degree=0, spread=0.1, scale_range=(0.002, 0.01), opacity_range=(0.02, 0.1))
    scene.positions[:, :2] += np.float32(0.1)  # inside one tile of the 48 x 48 view
    if bunched:  # 95% of the depths within 1e-3 of each other, the rest spread over 2 units
        far = rng.random(n) < 0.05
        scene.positions[:, 2] = np.where(far, rng.uniform(-1.0, 1.0, n), rng.uniform(0.0, 1e-3, n)).astype(np.float32)
    _compare_forward(scene, toy_camera(48, 48), np.ones(3), cuda)


def test_big_rectangles_binned_by_whole_ctas(cuda):
    """Primitives whose bounds cover more than 512 tiles (bin_big_kernel) next to small ones."""
    rng = np.random.default_rng(61)
    scene = random_scene(rng, 400, degree=1, spread=0.8, scale_range=(0.01, 0.05))
    scene.log_scales[:6] = np.log(np.float32(1.5))  # 6 huge footprints
    scene.opacity_raw[:6] = np.float32(-3.0)
    _compare_forward(scene, toy_camera(512, 384), np.ones(3), cuda)


@pytest.mark.parametrize("degree,views,n", [(3, 4, 400), (3, 19, 401), (0, 11, 401), (2, 19, 257)])
def test_multiview_deferred_colour_chain_matches_per_view(cuda, degree, views, n):
    """Several views of an SH set: the colour chain deferred into one kernel after the last
    view (bsr_backward_deferred_color + bsr_color_grad_views) gives the gradients of the
    per-view chain (bsr_backward per view) up to fp32 summation order.  Cases cover the
    view-chunk ring (> 2 chunks of 8), partial CTAs and coefficient runs that are not
    16 B multiples (degree 0 / 2)."""
    import torch

    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.training import TrainStep, render_targets

    rng = np.random.default_rng(71)
    tgt = PrimitiveSet.from_scene(random_scene(rng, 500, degree=degree))
    angles = np.linspace(-0.5, 0.7, views)
    cams = [toy_camera(64, 48, eye=(np.sin(a) * 4.0, 0.4 * np.cos(3 * a), -np.cos(a) * 4.0)) for a in angles]
    targets = render_targets(tgt, cams, np.ones(3))
    scene = random_scene(np.random.default_rng(72), n, degree=degree)
    a = TrainStep(PrimitiveSet.from_scene(scene), cams, targets, np.ones(3), defer_color=True)
    b = TrainStep(PrimitiveSet.from_scene(scene), cams, targets, np.ones(3), defer_color=False)
    assert a.drgb is not None and b.drgb is None
    a.step(check=True, adam=False)
    b.step(check=True, adam=False)
    torch.cuda.synchronize()
    for name in a.grads.groups:
        ga, gb = getattr(a.grads, name), getattr(b.grads, name)
        scale = max(float(gb.abs().max()), 1e-30)
        torch.testing.assert_close(ga, gb, rtol=1e-4, atol=1e-6 * scale, msg=name)
    np.testing.assert_allclose(a.loss_values.cpu().numpy(), b.loss_values.cpu().numpy(), rtol=1e-12)


@pytest.mark.parametrize("degree,views", [(3, 5), (1, 40)])
def test_public_api_multiview_accumulation_defers_colour_chain(cuda, degree, views):
    """render_backward(grads=g) over several views of an SH set defers each further view's
    colour chain into g (rasterizer._ColorPending) and applies them on the next read of
    g: the sums equal per-view fresh backwards added up (fp32 summation order), the 40-view
    case crosses the 32-view pending capacity, and a read between views flushes."""
    import torch

    from paper_2501_18630_b200 import PrimitiveSet, render_backward, render_tiled

    rng = np.random.default_rng(91)
    prims = PrimitiveSet.from_scene(random_scene(rng, 300, degree=degree))
    angles = np.linspace(-0.6, 0.6, views)
    cams = [toy_camera(64, 48, eye=(np.sin(a) * 4.0, 0.3 * np.cos(2 * a), -np.cos(a) * 4.0)) for a in angles]
    ups = [torch.as_tensor(rng.standard_normal((48, 64, 3)), dtype=torch.float32, device="cuda") for _ in cams]
    bg = np.ones(3)
    g = None
    for v, (cam, up) in enumerate(zip(cams, ups)):
        g = render_backward(prims, cam, bg, up, forward_out=render_tiled(prims, cam, bg), grads=g)
        if v == 2:
            assert g.__dict__.get("_pending") is not None and g.__dict__["_pending"].count == 2
            _ = g.positions  # a read applies the pending chains
            assert g.__dict__.get("_pending") is None
    ref = {name: torch.zeros_like(getattr(g, name)) for name in g.groups}
    for cam, up in zip(cams, ups):
        r = render_backward(prims, cam, bg, up, forward_out=render_tiled(prims, cam, bg))
        for name in ref:
            ref[name] += getattr(r, name)
    torch.cuda.synchronize()
    for name in g.groups:
        scale = max(float(ref[name].abs().max()), 1e-30)
        torch.testing.assert_close(getattr(g, name), ref[name], rtol=1e-4, atol=1e-6 * scale, msg=name)


def test_entry_capacity_overflow_retries(cuda):
    """A frame whose tile-entry capacity is too small reports BSR_ERR_CAPACITY with the
    entries needed; forward_raw grows the frame and the result is unchanged."""
    from paper_2501_18630_b200 import rasterizer as rz

    rng = np.random.default_rng(81)
    scene = random_scene(rng, 300, degree=1)
    cam = toy_camera(96, 64)
    rz._ENTRY_CAP[(300, 96, 64)] = 16  # far below the E this scene needs
    out, ref = _compare_forward(scene, cam, np.ones(3), cuda)
    assert out.frame.entry_cap >= ref["E"] > 16


def test_render_masked_matches_oracle(cuda):
    """rasterizer.py:214-227: render the primitives whose shape passes the predicate;
    contributions stay aligned with the full set (oracle on the kept subset)."""
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import rasterizer as rz

    rng = np.random.default_rng(90)
    scene = random_scene(rng, 300, degree=2)
    cam = toy_camera(80, 64)
    bg = np.array([1.0, 0.5, 0.25])
    pred = lambda b: b < np.float32(0.2)  # noqa: E731
    out = rz.render_masked(_gpu_prims(scene), cam, bg, pred)
    keep = np.nonzero(pred(scene.shapes))[0]
    assert 0 < keep.size < 300
    ref = orc.forward(scene.take(keep), cam, bg, core="c")
    assert np.abs(out.color.cpu().numpy() - ref["color"]).max() <= IMG_TOL
    full = np.zeros(300, np.int64)
    full[keep] = ref["contributions"]
    np.testing.assert_array_equal(out.contributions.cpu().numpy(), full)
    nothing = rz.render_masked(_gpu_prims(scene), cam, bg, lambda b: np.zeros(b.shape, bool))
    np.testing.assert_array_equal(nothing.color.cpu().numpy(), np.broadcast_to(bg.astype(np.float32), (64, 80, 3)))


def test_rasterize_autograd_matches_render_backward_and_oracle(cuda):
    """The torch.autograd entry (north star: PyTorch calling CUDA): gradients of
    sum(color * up) + sum(depth * upd) w.r.t. every input tensor equal render_backward's
    and the oracle's."""
    import torch

    from oracle import pipeline as orc
    from paper_2501_18630_b200 import rasterize

    rng = np.random.default_rng(91)
    scene = random_scene(rng, 200, degree=3)
    cam = toy_camera(72, 56)
    bg = np.array([0.3, 0.6, 0.9])
    up = rng.standard_normal((56, 72, 3))
    upd = rng.standard_normal((56, 72))
    leaves = [torch.tensor(np.asarray(getattr(scene, k)), device="cuda", requires_grad=True)
              for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh")]
    color, alpha, depth = rasterize(*leaves, cam, bg)
    fwd = orc.forward(scene, cam, bg, core="c")
    assert np.abs(color.detach().cpu().numpy() - fwd["color"]).max() <= IMG_TOL
    assert np.abs(alpha.cpu().numpy() - fwd["alpha"]).max() <= IMG_TOL
    loss = (color * torch.tensor(up, dtype=torch.float32, device="cuda")).sum() + \
        (depth * torch.tensor(upd, dtype=torch.float32, device="cuda")).sum()
    loss.backward()
    ref = orc.backward(scene, cam, bg, up, fwd, core="c", d_depth=upd)
    for name, t in zip(("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"), leaves):
        _grad_close(t.grad.cpu().numpy(), ref[name], name)


def test_render_tiled_async_status(cuda):
    """render_tiled does not synchronise once a shape's entry capacity is verified; a later
    overflow (scene grew) is reported by the asynchronous status check, and the next call
    re-verifies with a grown frame."""
    from paper_2501_18630_b200 import _lib
    from paper_2501_18630_b200 import rasterizer as rz

    rng = np.random.default_rng(92)
    scene = random_scene(rng, 500, degree=1)
    cam = toy_camera(96, 80)
    prims = _gpu_prims(scene)
    a = rz.render_tiled(prims, cam, np.ones(3))  # first call: synchronous check
    assert a.frame.pending is None
    b = rz.render_tiled(prims, cam, np.ones(3))  # verified shape: asynchronous
    assert b.frame.pending is not None
    info = b.frame.check()
    assert info["status"] == 0 and info["entries"] == a.frame.info["entries"]
    np.testing.assert_array_equal(a.color.cpu().numpy(), b.color.cpu().numpy())
    key = (500, 96, 80)
    rz._ENTRY_CAP[key] = 8  # pretend the verified capacity became too small
    c = rz.render_tiled(prims, cam, np.ones(3))
    with pytest.raises(_lib.CapacityError):
        rz.check_pending(block=True)
    assert key not in rz._VERIFIED and rz._ENTRY_CAP[key] >= info["entries"]
    d = rz.render_tiled(prims, cam, np.ones(3))  # re-verified synchronously, correct again
    assert d.frame.pending is None
    np.testing.assert_array_equal(a.color.cpu().numpy(), d.color.cpu().numpy())
    del c


def test_compat_drop_in_returns_reference_types(cuda):
    """compat.render_tiled / render_backward / render_masked: numpy in (a Spherical-Beta
    reference-layout set and an SH set), numpy fp64 / int64 out with the reference's
    field names, values equal to the device path's and the oracle's."""
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import compat
    from paper_2501_18630_b200.scenes import sb_random_scene

    rng = np.random.default_rng(93)
    cam = toy_camera(64, 48)
    bg = np.ones(3)
    for scene in (sb_random_scene(rng, 120).astype(np.float64), random_scene(rng, 120, degree=2)):
        out = compat.render_tiled(scene, cam, bg)
        assert out.color.dtype == np.float64 and out.contributions.dtype == np.int64
        ref = orc.forward(scene, cam, bg, core="c")
        np.testing.assert_array_equal(out.contributions, ref["contributions"])
        assert np.abs(out.color - ref["color"]).max() <= IMG_TOL
        assert np.abs(out.alpha - (1.0 - out.transmittance)).max() == 0.0
        up = rng.standard_normal((48, 64, 3))
        g = compat.render_backward(scene, cam, bg, up, forward_out=out)
        g2 = compat.render_backward(scene, cam, bg, up)  # recomputes the forward
        gref = orc.backward(scene, cam, bg, up, ref, core="c")
        for name, arr in g.parameters().items():
            _grad_close(arr, gref[name], name)
            _grad_close(getattr(g2, name), gref[name], name)
        m = compat.render_masked(scene, cam, bg, lambda b: b > 0)
        assert m.contributions.shape == (120,)


@pytest.mark.parametrize("case", ["random", "needles"])
def test_deterministic_backward_bitwise_and_parity(cuda, case):
    """bsr_backward_deterministic (bitwise determinism for a fixed input):
    two runs give bit-identical gradients; both match the oracle like the default mode."""
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import render_backward, render_tiled

    rng = np.random.default_rng(95)
    if case == "needles":
        scene, _ = _needle_scene(rng, 240)
        cam = toy_camera(256, 192)
    else:
        scene = random_scene(rng, 600, degree=3)
        cam = toy_camera(160, 120)
    bg = np.array([1.0, 0.9, 0.8])
    up = rng.standard_normal((cam.height, cam.width, 3))
    prims = _gpu_prims(scene)
    out = render_tiled(prims, cam, bg)
    a = render_backward(prims, cam, bg, up.astype(np.float32), forward_out=out, deterministic=True)
    b = render_backward(prims, cam, bg, up.astype(np.float32), forward_out=out, deterministic=True)
    assert torch_equal_bits(a.flat, b.flat)
    fwd = orc.forward(scene, cam, bg, core="c")
    ref = orc.backward(scene, cam, bg, up, fwd, core="c")
    for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"):
        _grad_close(getattr(a, k).cpu().numpy(), ref[k], k)


def torch_equal_bits(x, y):
    import torch

    return bool(torch.equal(x.view(torch.int32), y.view(torch.int32)))


def test_deterministic_training_steps_bitwise(cuda):
    """TrainStep(deterministic=True): a multi-view step (deferred colour chain) + Adam, ten
    times, gives bit-identical parameters in two independent runs."""
    import torch

    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.scenes import make_workload, target_scene
    from paper_2501_18630_b200.training import TrainStep, render_targets

    wl = make_workload("c3", seed=0, n=20_000, views=3, width=192, height=128)
    tgt = render_targets(PrimitiveSet.from_scene(target_scene("c3", 1, 20_000)), wl.cameras, wl.background)
    runs = []
    for _ in range(2):
        p = PrimitiveSet.from_scene(wl.scene)
        st = TrainStep(p, wl.cameras, tgt, wl.background, deterministic=True)
        st.step(check=True)
        for _ in range(9):
            st.step()
        torch.cuda.synchronize()
        runs.append((p.flat.clone(), st.loss_values.clone()))
    assert torch_equal_bits(runs[0][0], runs[1][0])
    assert torch.equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("degree", [3, 1, "sb"])
def test_precomputed_view_colours_are_bit_identical(cuda, degree):
    """bsr_view_colors + bsr_scene.view_rgb (multi-view steps read each view's colours from
    one pass over the SH coefficients) gives the same records as evaluating them in
    preprocess: identical loss values and, in the deterministic mode, bit-identical
    gradients and parameters after three Adam steps."""
    import torch

    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200.training import TrainStep, render_targets

    from paper_2501_18630_b200.scenes import sb_random_scene

    rng = np.random.default_rng(96)
    cams = [toy_camera(80, 64, eye=(np.sin(a) * 4.0, 0.5, -np.cos(a) * 4.0)) for a in np.linspace(-0.6, 0.6, 5)]
    if degree == "sb":  # the reference's Spherical-Beta colour
        mk = lambda r, n: PrimitiveSet.from_reference(sb_random_scene(r, n))  # noqa: E731
    else:
        mk = lambda r, n: PrimitiveSet.from_scene(random_scene(r, n, degree=degree))  # noqa: E731
    tgt = render_targets(mk(rng, 400), cams, np.ones(3))
    runs = []
    for pre in (True, False):
        p = mk(np.random.default_rng(97), 500)
        st = TrainStep(p, cams, tgt, np.ones(3), deterministic=True, precompute_colors=pre)
        assert (st.vrgb is not None) == pre
        st.step(check=True)
        for _ in range(2):
            st.step()
        torch.cuda.synchronize()
        runs.append((p.flat.clone(), st.loss_values.clone()))
    assert torch.equal(runs[0][1], runs[1][1])
    assert torch.equal(runs[0][0].view(torch.int32), runs[1][0].view(torch.int32))

def test_deferred_contributions_match_the_counting_forward(cuda):
    """render_tiled leaves the raster's part of the contributions to a count pass run on
    first access (bsr_contributions); it must equal the forward that counts inline, also
    when read after the backward and a parameter update (config-1 scene, flagged pixels
    included: their fp64 part is counted by the forward's replay either way)."""
    import torch

    from paper_2501_18630_b200 import PrimitiveSet, rasterizer as rz, training
    from paper_2501_18630_b200.scenes import make_workload

    wl = make_workload("c1", seed=3, n=100_000, views=1)
    prims = PrimitiveSet.from_scene(wl.scene)
    cam, bg = wl.cameras[0], wl.background
    # inline counting (defer_contributions = 0)
    h, w = cam.height, cam.width
    color = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
    ref = torch.zeros(len(prims), dtype=torch.int32, device="cuda")
    frame = rz.forward_raw(rz._prims_scene_c(prims), cam, bg, rz.outputs_c(color=color, contributions=ref),
                           contrib=ref, check=True)
    assert rz.frame_status(frame)["flagged_pixels"] > 0  # the replay's part is exercised
    out = rz.render_tiled(prims, cam, bg)
    assert torch.equal(out.color, color)
    g = rz.render_backward(prims, cam, bg, torch.ones_like(out.color), forward_out=out)
    state = training.AdamState(prims)
    training.adam_step(prims, g, state, training.group_lrs())  # parameters move; the frame does not
    got = out.contributions
    assert got.dtype == torch.int64
    np.testing.assert_array_equal(got.cpu().numpy(), ref.long().cpu().numpy())
    assert int(ref.sum()) > 0
    again = rz.render_tiled(prims, cam, bg)  # a second forward gets its own frame and count
    assert again.contributions.shape == got.shape
