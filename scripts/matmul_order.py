"""Which summation order does this image's numpy use for the projection matmuls?

The reference's EWA projection (primitive.py:221-277, restated in oracle/pipeline.py:project)
runs four float64 matmuls with inner dimension 3.  project.cuh's project64 must produce the
same bits; this script compares numpy's results with six candidate orders (exact FMA from
libm, compiled here with -ffp-contract=off) over seeded scene rows and prints the mismatch
count per order.  Measured (numpy 2.3 / scipy-openblas 0.3.30): the FMA chain
fma(x2, y2, fma(x1, y1, x0 y0)) matches every entry; the unfused ((x0 y0 + x1 y1) + x2 y2)
differs in 25-50% of them.
    python scripts/matmul_order.py
"""
import ctypes
import os
import subprocess
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import pipeline as orc  # noqa: E402
from paper_2501_18630_b200.scenes import make_workload  # noqa: E402

SRC = r"""
#include <math.h>
void orders(const double *a, const double *b, long n, double *out) {
  for (long i = 0; i < n; ++i) {
    const double *x = a + 3 * i, *y = b + 3 * i; double *o = out + 6 * i;
    o[0] = (x[0] * y[0] + x[1] * y[1]) + x[2] * y[2];
    o[1] = fma(x[2], y[2], fma(x[1], y[1], x[0] * y[0]));
    o[2] = fma(x[0], y[0], fma(x[1], y[1], x[2] * y[2]));
    o[3] = x[0] * y[0] + (x[1] * y[1] + x[2] * y[2]);
    o[4] = fma(x[2], y[2], x[0] * y[0] + x[1] * y[1]);
    o[5] = fma(x[0], y[0], x[1] * y[1]) + x[2] * y[2];
  }
}
"""
NAMES = ["unfused", "fma-chain", "fma-chain-rev", "unfused-rev", "fma-last", "fma-first"]


def main(n=100_000):
    d = tempfile.mkdtemp()
    with open(os.path.join(d, "o.c"), "w") as f:
        f.write(SRC)
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", os.path.join(d, "o.c"),
                           "-o", os.path.join(d, "libo.so"), "-lm"])
    lib = ctypes.CDLL(os.path.join(d, "libo.so"))

    def orders(a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty((len(a), 6))
        lib.orders(a.ctypes.data_as(ctypes.c_void_p), b.ctypes.data_as(ctypes.c_void_p), ctypes.c_long(len(a)),
                   out.ctypes.data_as(ctypes.c_void_p))
        return out

    def check(name, X, Y, Z):
        tot = np.zeros(6, np.int64)
        for i in range(X.shape[1]):
            for j in range(Y.shape[2]):
                o = orders(X[:, i, :], Y[:, :, j])
                tot += [(o[:, k] != Z[:, i, j]).sum() for k in range(6)]
        print(f"{name:14s} entries {Z.size:8d}  mismatches", dict(zip(NAMES, tot.tolist())))

    wl = make_workload("c2", seed=0)
    cam, sc = wl.cameras[0], wl.scene
    P = np.asarray(sc.positions, np.float64)[:n]
    t = P @ cam.rotation.T
    check("positions@R^T", P[:, None, :], np.broadcast_to(cam.rotation.T, (n, 3, 3)).copy(), t[:, None, :])
    scales = np.exp(np.asarray(sc.log_scales, np.float64))[:n]
    rs = orc.quat_to_rotation(np.asarray(sc.rotations)[:n]) * scales[..., None, :]
    sig = rs @ np.swapaxes(rs, -1, -2)
    check("rs@rs^T", rs, np.swapaxes(rs, -1, -2).copy(), sig)
    jac = orc.pinhole_jacobian(t + cam.translation, cam)
    a = jac @ cam.rotation
    check("J@R", jac, np.broadcast_to(cam.rotation, (n, 3, 3)).copy(), a)
    aS = a @ sig
    check("a@Sigma", a, sig, aS)
    check("(a@Sigma)@a^T", aS, np.swapaxes(a, -1, -2).copy(), aS @ np.swapaxes(a, -1, -2))


if __name__ == "__main__":
    main()
