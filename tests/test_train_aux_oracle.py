"""Pin the training-neighbour oracle (oracle/train_aux.py) against golden vectors that the
reference package itself produced (tests/golden/make_golden_train.py): MCMC relocation /
growth, position noise, loss regularisers, exponential_lr.  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import train_aux as ta

SB = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "base_colors", "lobe_axes", "lobe_colors")


@pytest.fixture(scope="module")
def g():
    return golden("train_aux.npz")


def _params(g, prefix):
    return {k: g[prefix + k].copy() for k in SB}


def test_numpy_choice_rule_is_cdf_searchsorted():
    # the draw rule the device reproduces: Generator.choice(a, size, p) with replace=True
    # consumes rng.random(size) and maps it through searchsorted(cumsum(p)/cdf[-1], side="right")
    rng = np.random.default_rng(5)
    w = rng.uniform(0.01, 1.0, 500)
    live = np.sort(rng.choice(5000, 500, replace=False))
    p = w / w.sum()
    a = np.random.default_rng(99).choice(live, size=2000, replace=True, p=p)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    b = live[np.searchsorted(cdf, np.random.default_rng(99).random(2000), side="right")]
    np.testing.assert_array_equal(a, b)


def test_find_dead_and_plan_match_reference(g):
    p = _params(g, "in_")
    dead = ta.find_dead(p["opacity_raw"])
    np.testing.assert_array_equal(dead, g["dead"])
    targets = ta.sample_live(p["opacity_raw"], g["u_plan"], exclude=dead)
    np.testing.assert_array_equal(targets, g["targets"])


def test_relocation_and_grow_match_reference(g):
    p = _params(g, "in_")
    m = {k: g["in_m_" + k].copy() for k in SB}
    v = {k: g["in_v_" + k].copy() for k in SB}
    ta.apply_relocation(p, [m, v], g["dead"], g["targets"])
    for k in SB:
        np.testing.assert_array_equal(p[k], g["reloc_" + k], err_msg=k)
    sources = ta.sample_live(p["opacity_raw"], g["u_grow"])
    grown, (gm, gv) = ta.grow(p, [m, v], sources)
    for k in SB:
        np.testing.assert_array_equal(grown[k], g["grow_" + k], err_msg=k)
        np.testing.assert_array_equal(gm[k], g["grow_m_" + k], err_msg=k)
        np.testing.assert_array_equal(gv[k], g["grow_v_" + k], err_msg=k)


def test_noise_matches_reference(g):
    p = _params(g, "in_")
    p["opacity_raw"] = g["noise_opacity_raw"]
    noise_lr, lr = g["noise_lr"]
    pos = ta.inject_noise(p, noise_lr, lr, g["noise_eta"])
    np.testing.assert_allclose(pos, g["noise_positions"], rtol=1e-13, atol=1e-15)
    assert np.abs(pos - p["positions"]).max() > 1e-6  # the noise actually moved something


def test_regularizers_match_reference(g):
    from oracle import pipeline as orc

    p = _params(g, "in_")
    v_img, _ = orc.loss(g["reg_a"], g["reg_b"])
    val, d_op, d_ls = ta.regularizers(p["opacity_raw"], p["log_scales"], 0.01, 0.01)
    assert v_img + val == pytest.approx(float(g["reg_value"]), rel=1e-12)
    np.testing.assert_allclose(d_op, g["reg_d_opacity_raw"], rtol=1e-14)
    np.testing.assert_allclose(d_ls, g["reg_d_log_scales"], rtol=1e-14)


def test_exponential_lr_matches_reference(g):
    for s, a, b in zip(g["lr_steps"], g["lr_plain"], g["lr_delay"]):
        assert ta.exponential_lr(int(s), 1.6e-4, 1.6e-6, 30000) == pytest.approx(a, rel=1e-15)
        assert ta.exponential_lr(int(s), 1.6e-4, 1.6e-6, 30000, 5000, 0.01) == pytest.approx(b, rel=1e-15)


def test_host_exponential_lr_matches_reference(g):
    # the library's schedule (evaluated by the same C code the device runs) on the host
    from paper_2501_18630_b200.training import exponential_lr

    for s, a, b in zip(g["lr_steps"], g["lr_plain"], g["lr_delay"]):
        assert exponential_lr(int(s), 1.6e-4, 1.6e-6, 30000) == pytest.approx(a, rel=1e-13)
        assert exponential_lr(int(s), 1.6e-4, 1.6e-6, 30000, 5000, 0.01) == pytest.approx(b, rel=1e-13)
