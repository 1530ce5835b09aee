"""project.cuh's dot3 restates numpy's float64 matmul (inner dimension 3) as the FMA chain
fma(x2, y2, fma(x1, y1, x0 y0)) that OpenBLAS's dgemm kernels compute; this pins that claim
on the oracle's own projection matmuls (oracle/pipeline.py:project, primitive.py:221-277)
so a numpy / BLAS change that moves the reference's bits shows up here, not as a rare
alpha-cutoff flip at full size."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))


@pytest.fixture(scope="module")
def mo():
    import shutil

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from scripts import matmul_order

    return matmul_order


def test_projection_matmuls_are_fma_chains(mo, capsys):
    mo.main(n=4000)
    out = capsys.readouterr().out
    lines = [ln for ln in out.splitlines() if "mismatches" in ln]
    assert len(lines) == 5
    for ln in lines:
        assert "'fma-chain': 0," in ln, ln
