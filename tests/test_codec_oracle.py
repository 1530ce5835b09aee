"""The codec restatement (oracle/codec.py) against the reference's own archives and arrays
(tests/golden/codec_*, codec.npz, written by the reference's compression.pack / unpack via
tests/golden/make_golden_train.py codec).  CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

CASES = [("codec_l2", 2, True), ("codec_l0_keep", 0, False)]


def _read(path):
    import cv2

    a = cv2.imread(path, cv2.IMREAD_UNCHANGED)
    if a.ndim == 3:  # OpenCV's BGR / BGRA -> RGB / RGBA
        a = a[:, :, [2, 1, 0, 3][: a.shape[2]]] if a.shape[2] == 4 else a[:, :, ::-1]
    return np.ascontiguousarray(a)


def _groups(g, name, lobes):
    p = lambda k: g[f"{name}_in_{k}"]
    out = [("opacity_raw", p("opacity_raw").reshape(-1, 1)), ("log_scales", p("log_scales")),
           ("rotations", p("rotations")), ("shapes", p("shapes").reshape(-1, 1)), ("base_colors", p("base_colors"))]
    for m in range(lobes):
        out += [(f"lobe{m}_axes", p("lobe_axes")[:, m]), (f"lobe{m}_colors", p("lobe_colors")[:, m])]
    return out


@pytest.mark.parametrize("name,lobes,sort", CASES)
def test_oracle_matches_reference_archive(name, lobes, sort):
    from oracle import codec

    g = golden("codec.npz")
    pos = g[f"{name}_in_positions"]
    np.testing.assert_array_equal(codec.morton_keys(pos), g[f"{name}_keys"])
    np.testing.assert_array_equal(codec.morton_order(pos), g[f"{name}_perm"])
    order = g[f"{name}_perm"] if sort else np.arange(len(pos))
    d = os.path.join(GOLDEN, name)
    man = json.load(open(os.path.join(d, "manifest.json")))
    rows, cols = man["grid"]
    assert (rows, cols) == codec.grid_dims(len(pos))
    for b, plane in enumerate(codec.position_planes(pos[order])):
        np.testing.assert_array_equal(_read(os.path.join(d, man["position_planes"][b])),
                                      codec.to_grid(plane, rows, cols))
    for gname, vals in _groups(g, name, lobes):
        codes, mins, maxs = codec.quantize(vals[order])
        spec = man["attributes"][gname]
        assert spec["min"] == [float(v) for v in mins] and spec["max"] == [float(v) for v in maxs]
        np.testing.assert_array_equal(_read(os.path.join(d, spec["file"])), codec.to_grid(codes, rows, cols))
        back = codec.dequantize(codes, mins, maxs)
        key = gname if not gname.startswith("lobe") else ("lobe_axes" if gname.endswith("axes") else "lobe_colors")
        ref = g[f"{name}_out_{key}"]
        if gname.startswith("lobe"):
            ref = ref[:, int(gname[4])]
        np.testing.assert_array_equal(back.reshape(ref.shape), ref)
    np.testing.assert_array_equal(codec.planes_to_positions(codec.position_planes(pos[order])),
                                  g[f"{name}_out_positions"])


def test_quantize_edges():
    from oracle import codec

    c, lo, hi = codec.quantize(np.array([[1.0, 2.0], [1.0, 4.0], [1.0, 3.0]]))
    assert c[:, 0].tolist() == [0, 0, 0] and c[:, 1].tolist() == [0, 255, 128]  # 127.5 -> even
    assert codec.dequantize(c, lo, hi)[:, 0].tolist() == [1.0, 1.0, 1.0]
    with pytest.raises(ValueError):
        codec.quantize(np.array([[np.nan]]))
