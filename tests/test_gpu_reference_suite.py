"""The reference's OWN rasterizer test-suite (pkg/tests/test_rasterizer.py, core-parametrised
through backend.get_core) run against the cuda core on the GPU box.

`make -C oracle refpkg` (run by __graft_entry__.build() where /root/reference exists)
places the unmodified reference package and its tests under oracle/_ref/pkg; that
directory travels to the GPU box with the snapshot.  tests/ref_core_plugin.py swaps the
core and applies fp32 float tolerances (see its docstring).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(REPO, "oracle", "_ref", "pkg")


@pytest.mark.parametrize("module", ["test_rasterizer.py"])
def test_reference_suite_on_cuda_core(cuda, module):
    path = os.path.join(PKG, "tests", module)
    if not os.path.exists(path):
        pytest.skip("reference package not built (make -C oracle refpkg)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([PKG, os.path.join(REPO, "tests"), REPO, env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", path, "-q", "-rA", "-p", "ref_core_plugin", "-p", "no:cacheprovider",
                        "--rootdir", PKG, "-o", "addopts="], cwd=PKG, env=env, capture_output=True, text=True,
                       timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    print(tail)
    assert r.returncode == 0, tail
    assert " passed" in r.stdout, tail
    # every core-parametrised test ran on the cuda core (and only on it)
    ran = [ln for ln in r.stdout.splitlines() if ln.startswith("PASSED")]
    assert sum("[cuda]" in ln for ln in ran) >= 15, tail
    assert not any("[compiled]" in ln or "[python]" in ln for ln in ran), tail


def test_reference_training_loop_switches_by_import(cuda):
    """betasplat.training.train with its renderer imported from paper_2501_18630_b200.compat
     trains the reference's toy scene like the reference's own
    renderer: same step count, best PSNR within 0.5 dB."""
    import json

    if not os.path.exists(os.path.join(PKG, "betasplat")):
        pytest.skip("reference package not built (make -C oracle refpkg)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([PKG, os.path.join(REPO, "tests"), REPO, env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, os.path.join(REPO, "tests", "ref_train_dropin.py")], cwd=REPO, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(res)
    ref, b2 = res["reference"], res["b200"]
    assert ref["steps"] == b2["steps"] > 0
    assert np.isfinite(b2["best_psnr"])
    assert abs(ref["best_psnr"] - b2["best_psnr"]) < 0.5, res
