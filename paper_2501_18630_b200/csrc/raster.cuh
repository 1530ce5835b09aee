// fp32 per-pair math shared by raster_fwd.cu and raster_bwd.cu.  Written with explicit
// round-to-nearest intrinsics so the compiler can neither contract nor reorder it: the
// backward recomputes alpha bit-identically to the forward, so both passes take exactly
// the same "alpha >= alpha_min" decisions.
#pragma once

#include "frame.cuh"

namespace bsr {

constexpr float kEps = 5.9604645e-08f;  // 2^-24

// 16-byte global -> shared copies (record gathers, double-buffered)
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct Pair {
    float dx, dy, r2, x, om, k, alpha;
};

// (1-x)^beta: two squarings for the Gaussian-like beta == 4 (no XU op); otherwise
// ex2(beta * lg2(1-x)) on the XU pipe.  Deterministic, shared by fwd/bwd.
__device__ __forceinline__ float beta_pow(float om, float beta) {
    if (beta == 4.0f) {
        const float o2 = __fmul_rn(om, om);
        return __fmul_rn(o2, o2);
    }
    return exp2f(__fmul_rn(beta, __log2f(om)));
}

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
    p.k = beta_pow(p.om, B.z);
    p.alpha = __fmul_rn(B.y, p.k);
    return p;
}

// fp64 evaluation for fp32-unsafe primitives (record kR < 0): r2 from the fp64 mean/conic
// side record (preprocess.cu), alpha in fp64, rounded once to fp32.  The fp32 conic form
// cancels catastrophically for extremely ill-conditioned footprints (near-plane
// primitives, condition numbers up to ~1e10); fp64 keeps their decisions certifiable.
__device__ __forceinline__ Pair eval_pair64(const double *m, const float4 B, int px, int py) {
    Pair p;
    const double dx = (double)px - m[0], dy = (double)py - m[1];
    const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(m[2], dx), dx),
                                          __dmul_rn(__dmul_rn(__dmul_rn(2.0, m[3]), dx), dy)),
                                __dmul_rn(__dmul_rn(m[4], dy), dy));
    const double x = fmin(fmax(r2, 0.0), 1.0);
    const double om = __dadd_rn(1.0, -x);
    double k;
    if (B.z == 4.0f) {
        const double o2 = __dmul_rn(om, om);
        k = __dmul_rn(o2, o2);
    } else {
        k = pow(om, (double)B.z);
    }
    p.dx = (float)dx;
    p.dy = (float)dy;
    p.r2 = (float)r2;
    p.x = (float)x;
    p.om = (float)om;
    p.k = (float)k;
    p.alpha = (float)__dmul_rn((double)B.y, k);
    return p;
}

// Relative error bound of the (1-x)^beta evaluation itself (inputs exact) + o * k rounding.
__device__ __forceinline__ float pow_rel_err(float beta) {
    // lg2.approx: <= 2^-22.6 abs on [0.5,2], 2 ulp of |lg2| <= 24 otherwise; ex2.approx 2 ulp;
    // beta*lg2 rounding: ln2 * |beta lg2| * eps  ->  <= (4 beta + 2) 1e-6 overall
    return beta == 4.0f ? 7.0f * kEps : (4.0f * fabsf(beta) + 2.0f) * 1.0e-6f + 3.0f * kEps;
}

// rcp.approx (relative error < 2^-22): only used inside error BOUNDS that carry a >= 1%
// safety factor, never in a value that is composited
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Record error word (Record.c.w, written by preprocess / the core seam):
//   Q = beta * kR + pow_rel_err(beta), rounded up, negative for fp32-unsafe primitives.
// The fp32 alpha of a sample with 1 - x = om then has relative error
//   <= beta kR / om + pow_rel_err(beta) <= Q / om        (om <= 1)
// (kR = r2 error bound of the primitive, propagated through (1-x)^beta).
__host__ __device__ inline float record_err_word(double kr, double beta, bool unsafe) {
    const double pe = beta == 4.0 ? 7.0 * 5.9604644775390625e-08
                                  : (4.0 * fabs(beta) + 2.0) * 1.0e-6 + 3.0 * 5.9604644775390625e-08;
    const float q = (float)((beta * kr + pe) * (1.0 + 1e-6));
    return unsafe ? -q : q;
}

// Same bound with the r2 error evaluated at this pixel instead of the footprint maximum
// (tighter; used on the rare alpha ~ alpha_min path):  |r2 error| <= eps (8 s + 3 (gx + gy)),
// s = sum of |terms| of the quadratic form, g = |grad r2 / 2| x (|d| + |mean - corner| + 1).
__device__ __forceinline__ float alpha_rel_err_pixel(const float4 A, const float4 B, const Pair &p) {
    const float s = fabsf(A.z * p.dx * p.dx) + fabsf(2.0f * A.w * p.dx * p.dy) + fabsf(B.x * p.dy * p.dy);
    const float gx = fabsf(A.z * p.dx + A.w * p.dy) * (fabsf(p.dx) + fabsf(A.x) + 1.0f);
    const float gy = fabsf(A.w * p.dx + B.x * p.dy) * (fabsf(p.dy) + fabsf(A.y) + 1.0f);
    const float dr2 = 1.5f * kEps * (8.0f * s + 3.0f * (gx + gy));
    return B.z * dr2 / fmaxf(p.om, 1e-30f) + pow_rel_err(B.z);
}

// Does the ellipse r2 < 1 (+ fp32 slack) of a primitive touch the pixel-centre rectangle
// [X0,X1] x [Y0,Y1]?  Exact minimum of the quadratic form over the rectangle (centre inside,
// else the minimum over the four edges), conservative by the record's r2 error bound.
__device__ __forceinline__ bool ellipse_hits_rect(const float4 A, const float4 B, const float4 C,
                                                  const int4 D, int X0, int X1, int Y0, int Y1,
                                                  float alpha_min) {
    if (D.y < X0 || D.x > X1 || D.w < Y0 || D.z > Y1) return false;
    const float mx = (float)D.x + A.x, my = (float)D.z + A.y;
    if (mx >= X0 && mx <= X1 && my >= Y0 && my <= Y1) return true;
    const float a = A.z, b = A.w, c = B.x;
    // approximate reciprocals only perturb the edge minimiser (second-order in q)
    const float ia = rcp_approx(a), ic = rcp_approx(c);
    float q = 3.0e38f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        // vertical edges x = X0 / X1
        const float dx = (float)(e ? X1 : X0) - mx;
        const float dy = fminf(fmaxf(my - b * dx * ic, (float)Y0), (float)Y1) - my;
        q = fminf(q, a * dx * dx + 2.0f * b * dx * dy + c * dy * dy);
        // horizontal edges y = Y0 / Y1
        const float ey = (float)(e ? Y1 : Y0) - my;
        const float ex = fminf(fmaxf(mx - b * ey * ia, (float)X0), (float)X1) - mx;
        q = fminf(q, a * ex * ex + 2.0f * b * ex * ey + c * ey * ey);
    }
    // a sample can only pass alpha >= alpha_min where r2 < x_max = 1 - (alpha_min / o)^(1/beta)
    // (o, beta as stored); relative slack 1e-4 covers the approximate lg2/ex2 and rounding
    if (B.y < alpha_min) return false;
    const float xmax = 1.0f - exp2f(__log2f(__fdividef(alpha_min, B.y)) * rcp_approx(B.z));
    // r2 slack 4 kR with kR <= |Q| / beta (record_err_word)
    return q < fminf(1.0f, xmax * 1.0001f + 1e-5f) + 4.04f * fabsf(C.w) * rcp_approx(B.z) + 1e-4f;
}

__device__ __forceinline__ bool bbox_hits_rect(const int4 D, int X0, int X1, int Y0, int Y1) {
    return !(D.y < X0 || D.x > X1 || D.w < Y0 || D.z > Y1);
}

}  // namespace bsr
