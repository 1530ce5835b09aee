"""Device codec (libbsr bsr_codec_*, compression.py) against the reference's own archives
(tests/golden/codec_*, codec.npz) and the oracle restatement (oracle/codec.py)."""

import filecmp
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu

CASES = [("codec_l2", 2, True), ("codec_l0_keep", 0, False)]
SB = ("positions", "opacity_raw", "rotations", "log_scales", "shapes", "base_colors", "lobe_axes", "lobe_colors")


def _prims(g, name):
    from paper_2501_18630_b200 import PrimitiveSet

    return PrimitiveSet(**{k: g[f"{name}_in_{k}"] for k in SB})


@pytest.mark.parametrize("name,lobes,sort", CASES)
def test_keys_and_order_match_reference(name, lobes, sort, cuda):
    from paper_2501_18630_b200 import compression

    g = golden("codec.npz")
    prims = _prims(g, name)
    keys = compression.morton_keys(prims.positions).cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(keys, g[f"{name}_keys"])
    np.testing.assert_array_equal(compression.sort_primitives(prims).cpu().numpy(), g[f"{name}_perm"])


@pytest.mark.parametrize("name,lobes,sort", CASES)
def test_pack_writes_the_reference_archive(name, lobes, sort, cuda, tmp_path):
    """Byte-identical archive: every PNG and the manifest."""
    from paper_2501_18630_b200 import compression

    g = golden("codec.npz")
    out = str(tmp_path / name)
    man = compression.pack(_prims(g, name), out, sort=sort)
    ref = os.path.join(GOLDEN, name)
    assert sorted(os.listdir(out)) == sorted(os.listdir(ref))
    for f in os.listdir(ref):
        assert filecmp.cmp(os.path.join(out, f), os.path.join(ref, f), shallow=False), f
    assert man == json.load(open(os.path.join(ref, "manifest.json")))
    assert compression.archive_size(out) == compression.archive_size(ref)


@pytest.mark.parametrize("name,lobes,sort", CASES)
def test_unpack_reads_the_reference_archive(name, lobes, sort, cuda):
    """Decoded values equal the reference's fp64 unpack rounded once to fp32."""
    from paper_2501_18630_b200 import compression

    g = golden("codec.npz")
    prims = compression.unpack(os.path.join(GOLDEN, name))
    assert prims.lobes == lobes and len(prims) == len(g[f"{name}_in_positions"])
    for k in SB:
        got = getattr(prims, k).cpu().numpy()
        np.testing.assert_array_equal(got, g[f"{name}_out_{k}"].astype(np.float32).reshape(got.shape), err_msg=k)


def test_sh_archive_roundtrip_and_reencode_stability(cuda, tmp_path):
    """SH extension: positions bit-exact, every other value within half a code step, and
    re-encoding a decoded archive reproduces its bytes (the lerp decode is exact at codes)."""
    import torch

    from paper_2501_18630_b200 import PrimitiveSet, compression
    from oracle import codec

    rng = np.random.default_rng(5)
    n, k = 3001, 16
    f = lambda a: np.asarray(a, np.float32)
    prims = PrimitiveSet(f(rng.normal(0, 3, (n, 3))), f(rng.normal(0, 1, (n, 4))), f(rng.normal(-3, 1, (n, 3))),
                         f(rng.normal(0, 1, n)), f(rng.normal(0, 1, n)), f(rng.normal(0, 0.3, (n, k, 3))))
    a = str(tmp_path / "a")
    man = compression.pack(prims, a)
    assert man["sh_coeffs"] == k and man["lobes"] == 0 and len(man["attributes"]) == 4 + k
    back = compression.unpack(a)
    perm = codec.morton_order(prims.positions.cpu().numpy().astype(np.float64))
    np.testing.assert_array_equal(back.positions.cpu().numpy(), prims.positions.cpu().numpy()[perm])
    for grp in ("opacity_raw", "log_scales", "rotations", "shapes", "sh"):
        src = getattr(prims, grp).cpu().numpy()[perm].reshape(n, -1).astype(np.float64)
        got = getattr(back, grp).cpu().numpy().reshape(n, -1).astype(np.float64)
        step = (src.max(0) - src.min(0)) / 255.0
        assert np.all(np.abs(got - src) <= 0.5 * step + 1e-6 * np.abs(src).max()), grp
    b = str(tmp_path / "b")
    compression.pack(back, b, sort=False)
    for fn in os.listdir(a):
        if fn.startswith("positions") or fn == "manifest.json":
            continue  # 'order' differs; planes compared above
        assert filecmp.cmp(os.path.join(a, fn), os.path.join(b, fn), shallow=False), fn
    torch.cuda.synchronize()


def test_large_sort_is_a_stable_permutation(cuda):
    """1M primitives with heavy key duplication: keys non-decreasing along perm, ties in
    ascending index (np.argsort(kind='stable')), against the oracle's keys."""
    import torch

    from paper_2501_18630_b200 import compression
    from oracle import codec

    rng = np.random.default_rng(9)
    n = 1 << 20
    pos = np.round(rng.uniform(-1, 1, (n, 3)) * 64) / 64  # coarse grid -> many equal keys
    pos = pos.astype(np.float32)
    keys = compression.morton_keys(torch.from_numpy(pos)).cpu().numpy().view(np.uint64)
    ref = codec.morton_keys(pos.astype(np.float64))
    np.testing.assert_array_equal(keys, ref)
    from paper_2501_18630_b200 import PrimitiveSet

    z = np.zeros((n, 1, 3), np.float32)
    prims = PrimitiveSet(pos, np.ones((n, 4), np.float32), np.zeros((n, 3), np.float32), np.zeros(n, np.float32),
                         np.zeros(n, np.float32), z)
    perm = compression.sort_primitives(prims).cpu().numpy()
    np.testing.assert_array_equal(perm, np.argsort(ref, kind="stable"))


def test_errors_match_reference(cuda, tmp_path):
    from paper_2501_18630_b200 import PrimitiveSet, compression

    with pytest.raises(compression.ArchiveError, match="no manifest"):
        compression.unpack(str(tmp_path))
    d = tmp_path / "v"
    d.mkdir()
    (d / "manifest.json").write_text(json.dumps({"version": 2}))
    with pytest.raises(compression.ArchiveError, match="unsupported archive version"):
        compression.unpack(str(d))
    rng = np.random.default_rng(1)
    n = 10
    bad = rng.normal(0, 1, (n, 3)).astype(np.float32)
    op = np.zeros(n, np.float32)
    op[3] = np.inf
    prims = PrimitiveSet(bad, np.ones((n, 4), np.float32), np.zeros((n, 3), np.float32), op, np.zeros(n, np.float32),
                         device="cuda", base_colors=np.zeros((n, 3), np.float32))
    with pytest.raises(ValueError, match="non-finite"):
        compression.pack(prims, str(tmp_path / "x"))
