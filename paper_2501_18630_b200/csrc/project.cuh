// fp64 projection + SH colour of one primitive.  Included ONLY by translation units
// compiled with -fmad=false (preprocess.cu, replay.cu) so that every caller produces the
// same bits, and so the operation order matches the reference's numpy arithmetic (ufuncs
// unfused, matmuls as OpenBLAS's FMA chains: dot3) as closely as a restatement can.
#pragma once

#include "common.cuh"

namespace bsr {

// primitive.py:28-35 (split-branch stable sigmoid)
__device__ __forceinline__ double sigmoid64(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

// kernel.py:42-44
__device__ __forceinline__ double shape_to_exponent64(double b) {
    return kBaseExponent * exp(fmin(fmax(b, -kShapeClamp), kShapeClamp));
}

// primitive.py:48-67 (normalised wxyz -> R)
__device__ __forceinline__ bool quat_to_rot64(const float *q4, double R[9]) {
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
    if (!(nrm >= 1e-12)) return false;
    w /= nrm;
    x /= nrm;
    y /= nrm;
    z /= nrm;
    R[0] = 1 - 2 * (y * y + z * z);
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = 1 - 2 * (x * x + z * z);
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = 1 - 2 * (x * x + y * y);
    return true;
}

// One entry of a numpy float64 matmul with inner dimension 3: OpenBLAS's dgemm kernels
// (this image's numpy, scipy-openblas 0.3.30) accumulate along k with FMAs,
// fma(x2, y2, fma(x1, y1, x0 y0)); measured bit-identical on every entry of the oracle's
// four projection matmuls (scripts/matmul_order.py), while the unfused sum differs in
// ~40% of entries -- enough, on near-singular covariances, to move an alpha across the
// 1/255 cutoff.
__device__ __forceinline__ double dot3(double x0, double x1, double x2, double y0, double y1, double y2) {
    return fma(x2, y2, fma(x1, y1, x0 * y0));
}

// numpy's float64 -> int32 cast on x86 (cvttsd2si): out-of-range / NaN -> INT32_MIN,
// followed by wrapping int32 arithmetic (primitive.py:254-261).
__device__ __forceinline__ int np_i32(double v) {
    return (v > -2147483649.0 && v < 2147483648.0) ? (int)v : (int)0x80000000;
}
__device__ __forceinline__ int np_i32_add(int a, int b) {
    return (int)((unsigned)a + (unsigned)b);
}

// primitive.py:221-277 for one primitive.
__device__ __forceinline__ Proj64 project64(const float *pos3, const float *quat4,
                                            const float *logs3, const KCam &cam) {
    Proj64 p;
    p.visible = false;
    p.degenerate = false;
    const double px = pos3[0], py = pos3[1], pz = pos3[2];
    const double *R = cam.R;
    // cam_pts = positions @ R^T + t
    p.tx = dot3(px, py, pz, R[0], R[1], R[2]) + cam.t[0];
    p.ty = dot3(px, py, pz, R[3], R[4], R[5]) + cam.t[1];
    p.tz = dot3(px, py, pz, R[6], R[7], R[8]) + cam.t[2];
    if (!(p.tz > kNearPlane)) return p;
    const double tx = p.tx, ty = p.ty, tz = p.tz;
    p.mx = cam.fx * tx / tz + cam.cx;
    p.my = cam.fy * ty / tz + cam.cy;
    // Sigma = (R diag s)(R diag s)^T
    double Q[9];
    if (!quat_to_rot64(quat4, Q)) {
        p.degenerate = true;
        return p;
    }
    const double s0 = exp((double)logs3[0]), s1 = exp((double)logs3[1]), s2 = exp((double)logs3[2]);
    double rs[9] = {Q[0] * s0, Q[1] * s1, Q[2] * s2, Q[3] * s0, Q[4] * s1,
                    Q[5] * s2, Q[6] * s0, Q[7] * s1, Q[8] * s2};
    double S[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            S[3 * i + j] = dot3(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], rs[3 * j], rs[3 * j + 1], rs[3 * j + 2]);
    // J (2x3), a = J @ R_cam (2x3)
    const double tz2 = tz * tz;
    const double j00 = cam.fx / tz, j02 = -cam.fx * tx / tz2;
    const double j11 = cam.fy / tz, j12 = -cam.fy * ty / tz2;
    double A[6];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        A[j] = dot3(j00, 0.0, j02, R[j], R[3 + j], R[6 + j]);
        A[3 + j] = dot3(0.0, j11, j12, R[j], R[3 + j], R[6 + j]);
    }
    // cov = (A @ S) @ A^T
    double AS[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            AS[3 * i + j] = dot3(A[3 * i], A[3 * i + 1], A[3 * i + 2], S[j], S[3 + j], S[6 + j]);
    double c00 = dot3(AS[0], AS[1], AS[2], A[0], A[1], A[2]);
    double c01 = dot3(AS[0], AS[1], AS[2], A[3], A[4], A[5]);
    double c11 = dot3(AS[3], AS[4], AS[5], A[3], A[4], A[5]);
    c00 += kCovConditioning;
    c11 += kCovConditioning;
    p.c00 = c00;
    p.c01 = c01;
    p.c11 = c11;
    const double det = c00 * c11 - c01 * c01;
    p.ca = c11 / det;
    p.cb = -c01 / det;
    p.cc = c00 / det;
    const double ex = sqrt(c00), ey = sqrt(c11);
    p.x0 = max(np_i32_add(np_i32(floor(p.mx - ex)), -kBoundsGuard), 0);
    p.x1 = min(np_i32_add(np_i32(ceil(p.mx + ex)), kBoundsGuard), cam.W - 1);
    p.y0 = max(np_i32_add(np_i32(floor(p.my - ey)), -kBoundsGuard), 0);
    p.y1 = min(np_i32_add(np_i32(ceil(p.my + ey)), kBoundsGuard), cam.H - 1);
    p.visible = (p.x0 <= p.x1) && (p.y0 <= p.y1);
    return p;
}

}  // namespace bsr
