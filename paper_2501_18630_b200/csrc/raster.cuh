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

// ---- sub-warp pixel groups -----------------------------------------------------------
// A warp owns an 8x4 pixel block.  With G groups the block splits into G sub-blocks
// (G = 1: 8x4, G = 2: two 4x4, G = 4: four 4x2) of 32/G lanes each; every group walks its
// own compacted entry list, so a warp-iteration evaluates G different entries and a pixel
// only visits entries whose support reaches its sub-block (tiny footprints: the 8x4 list
// is mostly entries that touch a few of its pixels).
template <int G>
struct SubBlock {
    static constexpr int lanes = 32 / G;
    static constexpr int w = G == 1 ? 8 : 4;
    static constexpr int h = G == 4 ? 2 : 4;
    __device__ static int group(int lane) { return lane / lanes; }
    __device__ static int ox(int q) { return G == 1 ? 0 : 4 * (q & 1); }
    __device__ static int oy(int q) { return G == 4 ? 2 * (q >> 1) : 0; }
    __device__ static int px(int lane) { return ox(group(lane)) + (lane % lanes) % w; }
    __device__ static int py(int lane) { return oy(group(lane)) + (lane % lanes) / w; }
    __device__ static unsigned mask(int q) { return G == 1 ? 0xffffffffu : (((1u << lanes) - 1u) << (q * lanes)); }
};

// Sub-block occupancy mask of one entry over a whole 16x16 tile (computed once per entry
// and batch by one thread, then read by every warp to build its groups' lists).  The tile
// is a grid of (16 / w) x (16 / h) sub-blocks, bit = row * (16 / w) + col; warp v's
// group q sits at col 2 (v & 1) + (q & 1) [G = 4] / 2 (v & 1) + q [G = 2] / v & 1 [G = 1],
// row 2 (v >> 1) + (q >> 1) [G = 4] / v >> 1.
//
// The test is exact per pixel row: for every pixel row y the ellipse {r2 <= xlim} (xlim =
// the alpha cutoff plus the record's r2 error slack, as in ellipse_hits_rect) spans
// dx in [(-b dy - sqrt(D)) / a, (-b dy + sqrt(D)) / a], D = a xlim - det dy^2; the span is
// padded for fp32 rounding (the D cancellation costs at most ~3e-4 of the half width) and
// clipped to the record bounds.  det = ac - b^2 of the record's fp32 conic is evaluated
// with Kahan's FMA scheme (accurate to ~1.5 ulp of det even for needle-like footprints,
// where the plain product difference cancels); fp32-unsafe records use the same spans
// with their larger r2 slack.  Non-positive-definite fp32 conics and the pair-counting
// variant (BBOX) use the bounds box.
template <int G>
struct TileGrid {
    static constexpr int w = SubBlock<G>::w, h = SubBlock<G>::h;
    static constexpr int cols = BSR_TILE / w, rows = BSR_TILE / h;
    __device__ static int bit(int warp, int q) {
        const int col = G == 4 ? 2 * (warp & 1) + (q & 1) : (G == 2 ? 2 * (warp & 1) + q : (warp & 1));
        const int row = G == 4 ? 2 * (warp >> 1) + (q >> 1) : (warp >> 1);
        return row * cols + col;
    }
};

// 32 x 32 bit transpose across a warp: lane r holds row r on entry; on exit lane c holds
// column c (bit r = bit c of row r).  Five butterfly stages of block swaps.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t m0 = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                          : s == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
        x = (lane & s) ? ((x & ~m0) | ((y & ~m0) >> s)) : ((x & m0) | ((y & m0) << s));
    }
    return x;
}

template <int G>
__device__ __forceinline__ uint32_t row_bits(int cx0, int cx1) {  // pixel columns (tile-relative)
    constexpr int w = TileGrid<G>::w;
    return ((2u << (cx1 / w)) - 1u) & ~((1u << (cx0 / w)) - 1u);
}

template <int G, bool BBOX>
__device__ __forceinline__ uint32_t entry_tile_mask(const float4 A, const float4 B, const float4 C, const int4 D,
                                                    int X0, int Y0, float alpha_min) {
    using TG = TileGrid<G>;
    // bounds box clipped to the tile (tile-relative pixel coordinates)
    const int bx0 = max(D.x - X0, 0), bx1 = min(D.y - X0, BSR_TILE - 1);
    const int by0 = max(D.z - Y0, 0), by1 = min(D.w - Y0, BSR_TILE - 1);
    if (bx0 > bx1 || by0 > by1) return 0u;
    if (!BBOX && B.y < alpha_min) return 0u;
    const float a = A.z, b = A.w, c = B.x;
    const float bb = __fmul_rn(b, b);
    const float det = __fadd_rn(__fmaf_rn(a, c, -bb), __fmaf_rn(-b, b, bb));  // Kahan 2x2
    if (BBOX || !(det > 0.f && a > 0.f)) {
        const uint32_t rb = row_bits<G>(bx0, bx1);
        uint32_t m = 0;
        for (int r = by0 / TG::h; r <= by1 / TG::h; ++r) m |= rb << (r * TG::cols);
        return m;
    }
    const float xmax = 1.0f - exp2f(__log2f(__fdividef(alpha_min, B.y)) * rcp_approx(B.z));
    const float xl = fminf(1.0f, xmax * 1.0001f + 1e-5f) + 4.04f * fabsf(C.w) * rcp_approx(B.z) + 1e-4f;
    const float ia = rcp_approx(a), id = rcp_approx(det);
    const float hy = sqrtf(xl * a * id) * 1.01f + 1e-3f;
    // fp32 error of a row span: sqrt of the D cancellation (<= 3.5e-4 sqrt(xl / a), the span
    // at dy = 0) plus a few ulp of the centre offset b dy / a
    const float pad0 = 1e-3f * sqrtf(xl * ia) + 2e-3f;
    // mean relative to the tile origin (exact: small integers plus the record's offset)
    const float mx = (float)(D.x - X0) + A.x, my = (float)(D.z - Y0) + A.y;
    const int y0 = max(by0, (int)ceilf(my - hy)), y1 = min(by1, (int)floorf(my + hy));
    uint32_t m = 0;
    for (int y = y0; y <= y1; ++y) {
        const float dy = (float)y - my;
        const float disc = fmaxf(a * xl - det * dy * dy, 0.f);
        const float off = b * dy * ia;
        const float half = sqrtf(disc) * ia * 1.001f + pad0 + 4e-7f * fabsf(off);
        const float cx = mx - off;
        const int x0 = max(bx0, (int)ceilf(cx - half)), x1 = min(bx1, (int)floorf(cx + half));
        if (x0 <= x1) m |= row_bits<G>(x0, x1) << ((y / TG::h) * TG::cols);
    }
    return m;
}

}  // namespace bsr
