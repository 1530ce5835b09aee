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
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Shared-memory loads through a 32-bit shared-window address computed once per kernel:
// indexing the double-buffered record arrays inside the pair lambdas made the compiler
// rebuild the shared window base (S2R SR_CgaCtaId + 6 uniform ops) on every pair.
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t addr) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

struct Pair {
    float dx, dy, u, w, r2, x, om, k, alpha;
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

// Cholesky factor of the conic Q = [[a, b], [b, c]] = L L^T, L = [[l11, 0], [l21, l22]]
// (fp64, host and device): the record carries (l11, l21, l22) instead of (a, b, c), and
//   r2 = a dx^2 + 2 b dx dy + c dy^2 = (l11 dx + l21 dy)^2 + (l22 dy)^2
// is evaluated as a sum of two squares.  The conic form's terms are ~condition-number
// times larger than r2 for elongated footprints and cancel; the factored form's error
// grows only with the square root of the condition number (chol_r2_error_bound), so far
// fewer primitives need the fp64 path.  Returns false if Q is not positive definite.
__host__ __device__ inline bool conic_cholesky(double a, double b, double c, double &l11, double &l21,
                                               double &l22) {
    l11 = l21 = l22 = 0.0;
    if (!(a > 0.0)) return false;
    l11 = sqrt(a);
    l21 = b / l11;
    const double d = c - l21 * l21;
    if (!(d > 0.0)) return false;
    l22 = sqrt(d);
    return true;
}

// Bound on |r2_fp32 - r2_exact| of eval_pair over a footprint |dx| <= X, |dy| <= Y with
// the mean stored relative to the bounds corner (|rel| <= X), where it matters (r2 <= ~1,
// so |u|, |w| <= ~1): rounding of the factors (eps U each) and of dx, dy (eps 2X, eps 2Y,
// times |d r2 / d dx| <= 2 l11, |d r2 / d dy| <= 2 (|l21| + l22)), and of the evaluation
// itself (u: eps (U + 1), w: eps, r2: 2 eps), U = l11 X + |l21| Y; safety factor 1.5.
__host__ __device__ inline double chol_r2_error_bound(double l11, double l21, double l22, double X, double Y) {
    const double U = l11 * X + fabs(l21) * Y;
    return 5.9604644775390625e-08 * 1.5 * (4.0 * U + 8.0 + 4.0 * l11 * X + 4.0 * (fabs(l21) + l22) * Y);
}

// Needles: primitives whose factored form still cancels (kR > kUnsafeR2Err: long thin
// footprints, r2 ~ 1 where l11 dx and l21 dy are each ~ l21 / l22 >> 1) but whose conic is
// positive definite.  They keep the fp32 path with compensated arithmetic: the frame's
// needle word holds (t_hi, t_lo) = l21 / l11 and the low parts of the mean offsets, dx and
// dy are formed exactly (TwoSum) as double-floats, and u = l11 (dx + t dy) is evaluated
// with one fused rounding on a small quantity.  What remains is rounding of the small
// terms themselves (bound below, X, Y the footprint half extents), so their decisions are
// certified like any other record's instead of running the fp64 evaluation per pixel.
__host__ __device__ inline double needle_r2_error_bound(double l11, double l21, double X, double Y) {
    const double t = fabs(l21 / l11);
    // |u| = l11 |s|, |w| <= 1 where it matters: du <= 4 eps |u| (s, l11, product), dw <= 3 eps |w|,
    // r2 = fma(w, w, u u): dr2 <= 8 eps u^2 + 6 eps w^2 + 2 eps r2 <= 10 eps, plus the neglected
    // second-order terms of the double-float parts (eps^2 t Y); safety factor 1.5
    return 5.9604644775390625e-08 * 1.5 * (12.0 + 8.0 * 5.9604644775390625e-08 * l11 * (X + t * Y));
}
// side word of a needle: (t_hi, t_lo, rel_x_lo, rel_y_lo); fp64-path records: (NaN, 1 if the
// fp64 conic has a factor (stored in side64) else 0, 0, 0)
__host__ __device__ inline float4 needle_word(double l11, double l21, double relx, double rely) {
    const double t = l21 / l11;
    const float th = (float)t, rx = (float)relx, ry = (float)rely;
    return make_float4(th, (float)(t - (double)th), (float)(relx - (double)rx), (float)(rely - (double)ry));
}

// _raster.pyx:107-113:  r2 = a dx^2 + 2 b dx dy + c dy^2 (factored, see conic_cholesky),
// x = clamp(r2, 0, 1), kernel = (1 - x)^beta, alpha = o * kernel.  px_rel / py_rel are
// pixel coordinates relative to the primitive's bounds corner (exact integers); the
// record holds A = (mean - corner, l11, l21), B.x = l22.
__device__ __forceinline__ Pair eval_pair(const float4 A, const float4 B, int px_rel, int py_rel) {
    Pair p;
    p.dx = __fsub_rn((float)px_rel, A.x);
    p.dy = __fsub_rn((float)py_rel, A.y);
    p.u = __fmaf_rn(A.w, p.dy, __fmul_rn(A.z, p.dx));
    p.w = __fmul_rn(B.x, p.dy);
    p.r2 = __fmaf_rn(p.w, p.w, __fmul_rn(p.u, p.u));
    p.x = fminf(fmaxf(p.r2, 0.0f), 1.0f);
    p.om = __fsub_rn(1.0f, p.x);
    p.k = beta_pow(p.om, B.z);
    p.alpha = __fmul_rn(B.y, p.k);
    return p;
}

// TwoSum: a + b = s + e exactly
__device__ __forceinline__ float two_sum(float a, float b, float &e) {
    const float s = __fadd_rn(a, b);
    const float bb = __fsub_rn(s, a);
    e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
    return s;
}

// The factor L (fp64) that the raster's whitened geometry partials of record c refer to
// (frame.cuh grad_acc: u = l11 dx + l21 dy, w = l22 dy):
//   fp32-safe records: the record's (l11, l21, l22);
//   needles: (l11, l11 t, l22) with t = t_hi + t_lo of the needle word (eval_needle's u);
//   fp64-path records with a positive-definite conic: the fp64 factor in side64;
// returns false for fp64-path records without one (xy-frame fp64 partials, add_geom64).
__device__ __forceinline__ bool record_factor64(const FrameView &f, uint32_t c, double &l11, double &l21,
                                                double &l22) {
    const Record &r = f.rec[c];
    const float4 ra = r.a, rb = r.b;
    if (!(r.c.w < 0.f)) {
        l11 = ra.z;
        l21 = ra.w;
        l22 = rb.x;
        return true;
    }
    const float4 N = f.needle[c];
    if (N.x == N.x) {
        l11 = ra.z;
        l21 = (double)ra.z * ((double)N.x + (double)N.y);
        l22 = rb.x;
        return true;
    }
    if (N.y != 0.f) {
        const double *s = f.side64 + (int64_t)kSide64 * c;
        l11 = s[0];
        l21 = s[1];
        l22 = s[2];
        return true;
    }
    return false;
}

// Compensated evaluation of a needle record (N = its needle word); same outputs as eval_pair.
__device__ __forceinline__ Pair eval_needle(const float4 A, const float4 B, const float4 N, int px_rel, int py_rel) {
    Pair p;
    float ex, ey;
    const float dxh = two_sum((float)px_rel, -A.x, ex), dyh = two_sum((float)py_rel, -A.y, ey);
    const float dxl = __fsub_rn(ex, N.z), dyl = __fsub_rn(ey, N.w);
    // s = dx + t dy: the large parts cancel inside one fused rounding, the rest are small
    const float s0 = __fmaf_rn(N.x, dyh, dxh);
    const float corr = __fmaf_rn(N.x, dyl, __fmaf_rn(N.y, dyh, dxl));
    const float sv = __fadd_rn(s0, corr);
    p.dx = __fadd_rn(dxh, dxl);
    p.dy = __fadd_rn(dyh, dyl);
    p.u = __fmul_rn(A.z, sv);
    p.w = __fmaf_rn(B.x, dyh, __fmul_rn(B.x, dyl));
    p.r2 = __fmaf_rn(p.w, p.w, __fmul_rn(p.u, p.u));
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
    p.u = p.w = 0.f;  // factored terms: fp32 path only
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
// (tighter; used on the rare alpha ~ alpha_min path), terms as in chol_r2_error_bound with
// this pixel's u, w, dx, dy.
__device__ __forceinline__ float alpha_rel_err_pixel(const float4 A, const float4 B, const Pair &p) {
    const float au = fabsf(p.u), aw = fabsf(p.w);
    const float U = fabsf(A.z * p.dx) + fabsf(A.w * p.dy);
    const float gx = 2.0f * fabsf(A.z) * au * (fabsf(p.dx) + fabsf(A.x) + 1.0f);
    const float gy = 2.0f * (fabsf(A.w) * au + fabsf(B.x) * aw) * (fabsf(p.dy) + fabsf(A.y) + 1.0f);
    const float dr2 = 1.5f * kEps * (4.0f * au * (U + au + 1.0f) + 6.0f * aw * aw + 2.0f * fabsf(p.r2) + gx + gy + 1.0f);
    return B.z * dr2 / fmaxf(p.om, 1e-30f) + pow_rel_err(B.z);
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
// x_max(o, beta) of the alpha cutoff, 1 - (alpha_min / o)^(1/beta), plus the record's r2
// error slack) spans dx in [(-l21 dy - sqrt(R)) / l11, (-l21 dy + sqrt(R)) / l11],
// R = xlim - (l22 dy)^2, in the factored form of the record; the span is padded for fp32
// rounding and clipped to the record bounds.  fp32-unsafe records use the same spans
// with their larger r2 slack; records without a positive factor and the pair-counting
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
                                                    int X0, int Y0, float alpha_min, int part = 0, int K = 1) {
    using TG = TileGrid<G>;
    // bounds box clipped to the tile (tile-relative pixel coordinates)
    const int bx0 = max(D.x - X0, 0), bx1 = min(D.y - X0, BSR_TILE - 1);
    const int by0 = max(D.z - Y0, 0), by1 = min(D.w - Y0, BSR_TILE - 1);
    if (bx0 > bx1 || by0 > by1) return 0u;
    if (!BBOX && B.y < alpha_min) return 0u;
    const float l11 = A.z, l21 = A.w, l22 = B.x;
    if (BBOX || !(l11 > 0.f && l22 > 0.f)) {
        if (part) return 0u;  // part 0 covers the whole box
        const uint32_t rb = row_bits<G>(bx0, bx1);
        uint32_t m = 0;
        for (int r = by0 / TG::h; r <= by1 / TG::h; ++r) m |= rb << (r * TG::cols);
        return m;
    }
    const float xmax = 1.0f - exp2f(__log2f(__fdividef(alpha_min, B.y)) * rcp_approx(B.z));
    const float xl = fminf(1.0f, xmax * 1.0001f + 1e-5f) + 4.04f * fabsf(C.w) * rcp_approx(B.z) + 1e-4f;
    const float sq = sqrtf(xl), il11 = rcp_approx(l11);
    const float hy = sq * rcp_approx(l22) * 1.01f + 1e-3f;
    // fp32 error of a row span: sqrt of the cancellation in xl - (l22 dy)^2 (<= 2.4e-4
    // sqrt(xl) / l11, the span at w = 0) plus a few ulp of the centre offset l21 dy / l11
    const float pad0 = 1e-3f * sq * il11 + 2e-3f;
    // mean relative to the tile origin (exact: small integers plus the record's offset)
    const float mx = (float)(D.x - X0) + A.x, my = (float)(D.z - Y0) + A.y;
    const int y0 = max(by0, (int)ceilf(my - hy)), y1 = min(by1, (int)floorf(my + hy));
    uint32_t m = 0;
    for (int y = y0 + part; y <= y1; y += K) {  // rows part, part + K, ... of the span
        const float dy = (float)y - my;
        const float wy = l22 * dy;
        const float rem = fmaxf(xl - wy * wy, 0.f);
        const float off = l21 * dy * il11;
        const float half = sqrtf(rem) * il11 * 1.001f + pad0 + 4e-7f * fabsf(off);
        const float cx = mx - off;
        const int x0 = max(bx0, (int)ceilf(cx - half)), x1 = min(bx1, (int)floorf(cx + half));
        if (x0 <= x1) m |= row_bits<G>(x0, x1) << ((y / TG::h) * TG::cols);
    }
    return m;
}

// Sub-block masks of a batch's nb entries, transposed into s_col[chunk][sub-block] (bit
// column per chunk of 32 entries).  With few entries (nb <= 128) K = 2..8 threads share an
// entry, each taking every K-th pixel row of its span, so the mask phase does not wait on
// single threads walking up to 16 rows; the parts are OR-combined (K | 32: an entry's
// parts sit in one warp) and regathered per chunk through s_mask.  Chunks >= ceil(nb / 32)
// of s_col are left untouched (never read).
// gmask (optional): the batch's slice of FrameView::emask, where each entry's mask is also
// stored for the backward.
template <int G, bool BBOX>
__device__ __forceinline__ void batch_masks(const Record *sr, int nb, int X0, int Y0, float alpha_min,
                                            uint32_t *s_mask, uint32_t (*s_col)[32], uint32_t *gmask = nullptr) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int K = 1;
    while (K < 8 && nb * K * 2 <= BSR_BLOCK) K <<= 1;
    if (K == 1) {
        uint32_t m = 0;
        if (t < nb) {
            const Record &r = sr[t];
            m = entry_tile_mask<G, BBOX>(r.a, r.b, r.c, r.d, X0, Y0, alpha_min);
            if (gmask) gmask[t] = m;
        }
        s_col[warp][lane] = warp_transpose32(m, lane);
        return;
    }
    const int e = t / K, part = t - e * K;
    uint32_t m = 0;
    if (e < nb) {
        const Record &r = sr[e];
        m = entry_tile_mask<G, BBOX>(r.a, r.b, r.c, r.d, X0, Y0, alpha_min, part, K);
    }
    for (int o = 1; o < K; o <<= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
    if (part == 0 && e < nb) {
        s_mask[e] = m;
        if (gmask) gmask[e] = m;
    }
    __syncthreads();
    if (warp < ((nb + 31) >> 5)) {
        const int ee = 32 * warp + lane;
        s_col[warp][lane] = warp_transpose32(ee < nb ? s_mask[ee] : 0u, lane);
    }
}

}  // namespace bsr
