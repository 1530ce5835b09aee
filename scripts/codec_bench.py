"""Codec measurement: device time of the Morton sort, the encode
(min/max + quantise + byte planes) and the decode on a c4-sized Spherical-Beta set, their
algorithmic bytes against the measured HBM peak, the end-to-end pack / unpack (PNG I/O on
the host included), and the oracle port (numpy) on a bounded sample of the same work.

    python scripts/codec_bench.py [--n 6000000] [--lobes 2]     -> one JSON line
"""
import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch


def events_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6_000_000)
    ap.add_argument("--lobes", type=int, default=2)
    ap.add_argument("--sample", type=int, default=1_000_000)
    args = ap.parse_args()
    from paper_2501_18630_b200 import PrimitiveSet, _lib, compression
    from paper_2501_18630_b200.compression import _groups_c, _scratch, attribute_groups, grid_dims

    n, m = args.n, args.lobes
    rng = np.random.default_rng(0)
    f = lambda a: np.asarray(a, np.float32)
    prims = PrimitiveSet(f(rng.normal(0, 2, (n, 3))), f(rng.normal(0, 1, (n, 4))), f(rng.normal(-4, 1, (n, 3))),
                         f(rng.normal(0, 1, n)), f(rng.normal(0, 1, n)), device="cuda",
                         base_colors=f(rng.normal(0, 1, (n, 3))), lobe_axes=f(rng.normal(0, 1, (n, m, 3))),
                         lobe_colors=f(rng.normal(0, 1, (n, m, 3))))
    lib = _lib.load()
    st = ctypes_stream = __import__("ctypes").c_void_p(torch.cuda.current_stream().cuda_stream)
    rows, cols = grid_dims(n)
    cells = rows * cols
    groups = attribute_groups(n, None, m)
    gc = _groups_c(groups)
    ch = sum(g[3] for g in groups)
    scratch, nbytes = _scratch(n, prims.flat.device)
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    planes = torch.empty(12 * cells, dtype=torch.uint8, device="cuda")
    codes = torch.empty(cells * ch, dtype=torch.uint8, device="cuda")
    mm = torch.empty((2, ch), dtype=torch.float64, device="cuda")
    flat2 = torch.empty_like(prims.flat)
    pos2 = torch.empty(n * 3, dtype=torch.float32, device="cuda")

    def sort():
        lib.bsr_codec_sort(prims.positions.data_ptr(), n, None, perm.data_ptr(), scratch.data_ptr(), nbytes, st)

    def encode():
        lib.bsr_codec_encode(prims.flat.data_ptr(), prims.positions.data_ptr(), n, perm.data_ptr(), len(groups), gc,
                             rows, cols, planes.data_ptr(), codes.data_ptr(), mm[0].data_ptr(), mm[1].data_ptr(),
                             None, scratch.data_ptr(), nbytes, st)

    def decode():
        lib.bsr_codec_decode(planes.data_ptr(), codes.data_ptr(), mm[0].data_ptr(), mm[1].data_ptr(), n, len(groups),
                             gc, rows, cols, flat2.data_ptr(), pos2.data_ptr(), st)

    t_sort, t_enc, t_dec = events_ms(sort), events_ms(encode), events_ms(decode)
    params = 12 + 4 * ch  # floats read per primitive: positions + quantised channels
    # algorithmic bytes: sort = key build (read 12 B, write 12 B) + 8 radix passes over
    # (key 8 B + value 4 B) read + write + perm write; encode = min/max read + gather read +
    # 4 planes x 3 B + ch code bytes written (+ perm read); decode = inverse
    b_sort = n * (24 + 8 * 24 + 12)
    b_enc = n * (4 * ch + params + 8) + cells * (12 + ch)
    b_dec = cells * 0 + n * (12 + ch) + n * params
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = next((v for k, v in peaks.items() if "hbm" in k.lower() and isinstance(v, (int, float))), None)

    # end to end through the public API (PNG encode / decode on the host)
    with tempfile.TemporaryDirectory() as d:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        compression.pack(prims, d)
        t_pack = time.perf_counter() - t0
        t0 = time.perf_counter()
        back = compression.unpack(d)
        torch.cuda.synchronize()
        t_unpack = time.perf_counter() - t0
        size = compression.archive_size(d)
    del back
    # oracle port (numpy) on a bounded sample of the device work: keys + sort + quantise
    from oracle import codec

    s = min(args.sample, n)
    host = {g: getattr(prims, g)[:s].cpu().numpy().astype(np.float64) for g in prims.groups}
    t0 = time.perf_counter()
    order = codec.morton_order(host["positions"])
    for name, start, stride, c in groups:
        base = {"opacity_raw": "opacity_raw", "log_scales": "log_scales", "rotations": "rotations",
                "shapes": "shapes", "base_colors": "base_colors"}.get(name)
        vals = host[base] if base else host["lobe_axes" if name.endswith("axes") else "lobe_colors"][:, int(name[4])]
        codec.quantize(vals[order])
    codec.position_planes(host["positions"][order])
    t_cpu = time.perf_counter() - t0
    line = {"metric": "codec_encode_throughput", "unit": "Mprims/s", "n": n, "lobes": m,
            "value": n / ((t_sort + t_enc) * 1e-3) / 1e6,
            "stages_ms": {"sort": t_sort, "encode": t_enc, "decode": t_dec},
            "hbm_gbs": {"sort": b_sort / t_sort / 1e6, "encode": b_enc / t_enc / 1e6, "decode": b_dec / t_dec / 1e6},
            "hbm_peak_gbs": peak,
            "e2e_s": {"pack": t_pack, "unpack": t_unpack, "archive_bytes": size},
            "cpu_baseline": {"kind": "port", "cores": 1, "sample": f"{s} primitives (keys + stable sort + quantise + planes)",
                             "value": s / t_cpu / 1e6, "unit": "Mprims/s"}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
