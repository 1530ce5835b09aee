// fp32 per-pair math shared by raster_fwd.cu and raster_bwd.cu.  Written with explicit
// round-to-nearest intrinsics so the compiler can neither contract nor reorder it: the
// backward recomputes alpha bit-identically to the forward, so both passes take exactly
// the same "alpha >= alpha_min" decisions.
#pragma once

#include "frame.cuh"

namespace bsr {

struct Pair {
    float dx, dy, r2, x, om, k, alpha;
};

// _raster.pyx:107-113:  r2 = a dx^2 + 2 b dx dy + c dy^2, x = clamp(r2, 0, 1),
// kernel = (1 - x)^beta, alpha = o * kernel.  px_rel / py_rel are pixel coordinates
// relative to the primitive's bounds corner (exact integers).
__device__ __forceinline__ Pair eval_pair(const float4 A, const float4 B, int px_rel, int py_rel) {
    Pair p;
    p.dx = __fsub_rn((float)px_rel, A.x);
    p.dy = __fsub_rn((float)py_rel, A.y);
    float t = __fmul_rn(B.x, __fmul_rn(p.dy, p.dy));
    t = __fmaf_rn(__fmul_rn(__fmul_rn(2.0f, A.w), p.dx), p.dy, t);
    p.r2 = __fmaf_rn(__fmul_rn(A.z, p.dx), p.dx, t);
    p.x = fminf(fmaxf(p.r2, 0.0f), 1.0f);
    p.om = __fsub_rn(1.0f, p.x);
    if (B.z == 4.0f) {
        const float o2 = __fmul_rn(p.om, p.om);
        p.k = __fmul_rn(o2, o2);
    } else {
        p.k = powf(p.om, B.z);
    }
    p.alpha = __fmul_rn(B.y, p.k);
    return p;
}

// Conservative bound on the relative error of the fp32 alpha versus the exact (fp64)
// evaluation of the same primitive (record rounding, dx/dy rounding through the stored
// mean, r2 evaluation, the (1-x)^beta evaluation).  Only evaluated on rare paths.
__device__ __forceinline__ float alpha_rel_err(const float4 A, const float4 B, const Pair &p) {
    const float eps = 5.9604645e-08f;  // 2^-24
    const float s = fabsf(A.z * p.dx * p.dx) + fabsf(2.0f * A.w * p.dx * p.dy) +
                    fabsf(B.x * p.dy * p.dy);
    const float gx = fabsf(A.z * p.dx + A.w * p.dy) * (fabsf(p.dx) + fabsf(A.x) + 1.0f);
    const float gy = fabsf(A.w * p.dx + B.x * p.dy) * (fabsf(p.dy) + fabsf(A.y) + 1.0f);
    const float dr2 = eps * (8.0f * s + 3.0f * (gx + gy));
    const float beta = B.z;
    const float pow_err = (beta == 4.0f) ? 4.0f * eps : 4.0f * eps * (1.0f + fabsf(beta * __logf(fmaxf(p.om, 1e-30f))));
    return beta * dr2 / fmaxf(p.om, 1e-30f) + pow_err + 3.0f * eps;
}

}  // namespace bsr
