"""Pin the oracle before trusting it (CPU only).

1. oracle/raster_oracle.c (our C restatement) is bit-identical to the reference's own
   compiled core (oracle/_ref, built from /root/reference .../_raster.pyx) on raw, T and
   contributions -- skipped only where that build is absent.
2. oracle/pipeline.py (numpy restatement + SH adapter) reproduces the golden vectors that
   tests/golden/make_golden.py produced by running the reference package itself.
3. Per-pixel counts (not produced by the reference) sum to the reference's contributions.
"""

import numpy as np
import pytest

from conftest import golden, golden_scene_camera

from oracle import pipeline as orc


def _fwd(g, core="c"):
    scene, cam = golden_scene_camera(g)
    return scene, cam, orc.forward(scene, cam, g["bg"], core=core, threads=4)


@pytest.mark.parametrize("name", ["c0_forward.npz", "sh3_fwd_bwd.npz", "shapes_sh2.npz"])
def test_forward_matches_reference_golden(name):
    g = golden(name)
    _, _, out = _fwd(g)
    np.testing.assert_array_equal(out["offsets"], g["offsets"])
    np.testing.assert_array_equal(out["lists"], g["lists"])
    np.testing.assert_array_equal(out["contributions"], g["contributions"])
    # same numpy ops, same C expression order -> exact
    np.testing.assert_array_equal(out["raw"], g["raw"])
    np.testing.assert_array_equal(out["T"], g["T"])
    if "order" in g:
        np.testing.assert_array_equal(out["order"], g["order"])
        np.testing.assert_array_equal(out["batch"]["indices"], g["indices"])


def test_c0_golden_intermediates():
    g = golden("c0_forward.npz")
    _, _, out = _fwd(g)
    s = out["shaded"]["sorted"]
    np.testing.assert_array_equal(s["bounds"], g["bounds"])
    np.testing.assert_array_equal(s["depths"], g["depths"])
    np.testing.assert_allclose(s["colors"], g["colors"], rtol=0, atol=1e-15)


def test_pixel_counts_sum_to_contributions():
    g = golden("c0_forward.npz")
    _, _, out = _fwd(g)
    assert int(out["pix_count"].sum()) == int(out["contributions"].sum())
    # last entry is inside the pixel's tile list, or -1 for no contributor
    assert ((out["pix_last"] >= 0) == (out["pix_count"] > 0)).all()


@pytest.mark.skipif(not orc.have_ref_core(), reason="reference core not built here")
@pytest.mark.parametrize("name", ["sh3_fwd_bwd.npz", "shapes_sh2.npz"])
def test_c_core_bit_identical_to_reference_core(name):
    g = golden(name)
    scene, cam = golden_scene_camera(g)
    _, order, shaded = orc.view_setup(scene, cam)
    s = shaded["sorted"]
    off, lists = orc.tile_bins(s["bounds"], cam.height, cam.width)
    a = orc.raster_forward(s, cam.height, cam.width, g["bg"], off, lists, core="c", threads=3)
    b = orc.raster_forward(s, cam.height, cam.width, g["bg"], off, lists, core="ref", threads=2)
    for k in ("raw", "T", "contrib"):
        np.testing.assert_array_equal(a[k], b[k])
    d_raw = np.where(a["raw"] >= 0, g["upstream"], 0.0)
    ga = orc.raster_backward(s, cam.height, cam.width, g["bg"], a["raw"], d_raw, off, lists, core="c")
    gb = orc.raster_backward(s, cam.height, cam.width, g["bg"], b["raw"], d_raw, off, lists, core="ref")
    for x, y in zip(ga[:5], gb[:5]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("name", ["sh3_fwd_bwd.npz", "shapes_sh2.npz"])
def test_backward_matches_reference_golden(name):
    g = golden(name)
    scene, cam, out = _fwd(g)
    grads = orc.backward(scene, cam, g["bg"], g["upstream"], out, core="c", threads=4)
    for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "sh"):
        ref = g["g_" + k]
        scale = max(np.abs(ref).max(), 1e-30)
        np.testing.assert_allclose(grads[k], ref, rtol=1e-10, atol=1e-12 * scale, err_msg=k)


def test_loss_matches_reference_golden():
    g = golden("loss.npz")
    value, d_image = orc.loss(g["a"], g["b"])
    assert value == pytest.approx(float(g["value"]), rel=1e-13)
    np.testing.assert_allclose(d_image, g["d_image"], rtol=1e-10, atol=1e-16)
    sv, sg = orc.ssim(g["a"], g["b"])
    assert sv == pytest.approx(float(g["ssim"]), rel=1e-13)


def test_ssim_identity_is_one():
    # tests/test_training.py:34-40 of the reference
    a = np.random.default_rng(0).uniform(0, 1, (20, 24, 3))
    v, _ = orc.ssim(a, a)
    assert v == pytest.approx(1.0, abs=1e-12)


def test_adam_matches_reference_golden():
    g = golden("adam.npz")
    names = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "base_colors")
    p = {k: g["p0_" + k].copy() for k in names}
    m = {k: np.zeros_like(v) for k, v in p.items()}
    v = {k: np.zeros_like(x) for k, x in p.items()}
    lrs = {k: (1.6e-4 if k == "positions" else 5e-3) for k in names}
    for i in range(3):
        orc.adam_step(p, {k: g[f"g{i}_" + k] for k in names}, m, v, i + 1, lrs)
    for k in names:
        np.testing.assert_allclose(p[k], g["p3_" + k], rtol=0, atol=1e-15)


def test_single_primitive_center_pixel_closed_form():
    """tests/test_rasterizer.py:50-66: centre pixel = o*c + (1-o)*bg."""
    from paper_2501_18630_b200.scenes import SplatScene
    from conftest import toy_camera

    cam = toy_camera(33, 33)
    o = 0.6
    base = np.array([0.8, 0.3, 0.1])
    scene = SplatScene(positions=np.zeros((1, 3)), rotations=np.array([[1.0, 0, 0, 0]]),
                       log_scales=np.log(np.full((1, 3), 0.25)),
                       opacity_raw=np.array([np.log(o) - np.log1p(-o)]), shapes=np.zeros(1),
                       sh=(base / orc._C0)[None, None, :])
    out = orc.forward(scene, cam, np.ones(3))
    np.testing.assert_allclose(out["color"][16, 16], base * o + (1 - o), atol=1e-9)


def test_bounds_worked_example():
    """tests/test_primitive.py:157-159: mean (10, 10), cov diag(4, 9) -> (7, 13, 6, 14)."""
    mean, ex, ey, w, h = np.array([10.0, 10.0]), 2.0, 3.0, 100, 100
    x0 = max(int(np.floor(mean[0] - ex)) - orc.BOUNDS_GUARD, 0)
    x1 = min(int(np.ceil(mean[0] + ex)) + orc.BOUNDS_GUARD, w - 1)
    y0 = max(int(np.floor(mean[1] - ey)) - orc.BOUNDS_GUARD, 0)
    y1 = min(int(np.ceil(mean[1] + ey)) + orc.BOUNDS_GUARD, h - 1)
    assert (x0, x1, y0, y1) == (7, 13, 6, 14)


@pytest.mark.parametrize("name", ["sb_small.npz", "sb_medium.npz"])
def test_spherical_beta_matches_unmodified_reference(name):
    """The oracle's Spherical-Beta path == the reference's own render_tiled / render_backward."""
    g = golden(name)
    scene, cam = golden_scene_camera(g)
    out = orc.forward(scene, cam, g["bg"], core="c", threads=3)
    np.testing.assert_array_equal(out["contributions"], g["contributions"])
    np.testing.assert_array_equal(out["raw"], g["raw"])
    grads = orc.backward(scene, cam, g["bg"], g["upstream"], out, core="c", threads=3)
    for k in ("positions", "rotations", "log_scales", "opacity_raw", "shapes", "base_colors", "lobe_axes",
              "lobe_colors"):
        ref = g["g_" + k]
        scale = max(np.abs(ref).max(), 1e-30)
        np.testing.assert_allclose(grads[k], ref, rtol=1e-10, atol=1e-12 * scale, err_msg=k)
