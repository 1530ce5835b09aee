"""pytest plugin: run the REFERENCE's own core-parametrised tests against the cuda core.

Loaded by tests/test_gpu_reference_suite.py as
    python -m pytest oracle/_ref/pkg/tests/test_rasterizer.py -p ref_core_plugin
with PYTHONPATH = oracle/_ref/pkg (the reference package, built by `make -C oracle
refpkg`) + tests/ + the repo root.  It

  * makes betasplat.backend offer one core, "cuda" = paper_2501_18630_b200.cuda_core
    (the core plugin seam, backend.py:28-42), so the reference's ``core`` fixture
    (tests/conftest.py:34-36) parametrises every test over it;
  * floors numpy.testing.assert_allclose's atol at FP32_ATOL for float data: the cuda core
    composites in fp32, the reference tests assert fp64 agreement (1e-9 .. 1e-12) against
    fp64 per-pixel oracles ("tests asserting 1e-10 on floats need fp32
    tolerances; integer checks stay exact"); assert_array_equal is untouched, so every
    bit-identity test (storage order, thread count, tiled == naive on one tile, masks,
    zero gradients, contributions) stays exact;
  * marks the two finite-difference tests xfail: central differences of an fp32 image
    with h = 1e-5 / 1e-6 carry ~1e-1 relative noise whatever the core computes (measured
    on the B200: 13% on test_matches_finite_differences); the analytic gradients they
    would check are compared with the reference's fp64 analytic gradients instead
    (tests/test_gpu_parity.py, tests/test_gpu_fullsize.py), and the reference's own FD
    tests pin those fp64 gradients.
"""

import numpy as np
import pytest

FP32_ATOL = 1e-5  # images: 10x inside the north star's 1e-4
FD_TESTS = ("test_matches_finite_differences", "test_directional_derivative_matches")


def _install():
    """Patch at import time: ``-p`` plugins are imported before the reference's initial
    conftest, whose ``core`` fixture evaluates backend.available_backends() on import."""
    from betasplat import backend

    from paper_2501_18630_b200 import cuda_core

    orig = backend.get_core
    backend.available_backends = lambda: ["cuda"]

    def get_core(name=None):
        return cuda_core if name == "cuda" else orig(name)

    backend.get_core = get_core

    allclose = np.testing.assert_allclose

    def assert_allclose_fp32(actual, desired, rtol=1e-7, atol=0, *args, **kwargs):
        if np.asarray(desired).dtype.kind == "f":
            atol = max(atol, FP32_ATOL)
        return allclose(actual, desired, rtol, atol, *args, **kwargs)

    np.testing.assert_allclose = assert_allclose_fp32


_install()


def pytest_collection_modifyitems(config, items):
    for it in items:
        if it.originalname in FD_TESTS:
            it.add_marker(pytest.mark.xfail(reason="fp64 central differences of an fp32 render (noise ~1e-1)",
                                            strict=True))
