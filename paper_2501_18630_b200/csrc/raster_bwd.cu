// K5 raster_bwd: analytic gradients of the composite (_raster.pyx:158-287).
//
// Same CTA-per-tile layout as the forward, but each pixel walks its tile list
// BACK-TO-FRONT from its own last contributor (saved by the forward), recovering
// T_k = T_{k+1} / (1 - alpha_k) and carrying the normalised "behind" colour
//     B_{k-1} = alpha_k c_k + (1 - alpha_k) B_k,   B_last = background,
// so that  dL/dalpha_k = T_k [ g.(c_k - B_k) + g_D (z_k - B^D_k) ]  equals the
// reference's  g.c T - g.behind / (1 - alpha)  without the raw - prefix cancellation.
// alpha is recomputed with the forward's exact fp32 code (raster.cuh), so the
// alpha >= alpha_min decisions are the forward's.  Pixels the forward handed to the fp64
// replay have last == 0 here and are differentiated by replay.cu instead.
//
// Per batch each warp builds the compacted list of entries whose ellipse reaches its 8x4
// block and that precede the warp's furthest last contributor, then walks it backwards.
// Per pair the 11 partials (d mean2d x2, d conic x3, d opacity, d beta, d rgb x3, d z)
// are reduced across the warp with a 16-shuffle transpose reduction and added with one
// warp-wide RED instruction per (warp, entry) into grad_acc[compact][12].
#include <stdlib.h>

#include "raster.cuh"

namespace bsr {

struct RasterBwdArgs {
    FrameView f;
    const float *d_color;  // (H,W,3) dL/d colour (dL/d raw when use_mask is false)
    bool use_mask;         // clamp chain d_raw = d_color * [raw >= 0] (rasterizer.py:253)
    const float *d_depth;  // (H,W) or nullptr
    float bg[3];
    float alpha_min;
    const uint32_t *lists;
    const uint2 *ranges;
    const Record *rec;
    unsigned long long *stats;  // optional: [2] evaluated pairs
    int direct_max;
};

// fp64 pair evaluation + the two conic-gradient terms for fp32-unsafe primitives; kept
// out of line so the common fp32 path is not if-converted into predicated fp64 code.
// Returned by value (no pointer arguments: those would force the caller's ga/gb into
// local memory on the hot path).
struct PairG {
    Pair p;
    float ga, gb;
};
__device__ __noinline__ PairG unsafe_pair_bwd(const double *m64, float4 B, int px, int py) {
    const double dx = (double)px - m64[0], dy = (double)py - m64[1];
    PairG r;
    r.ga = (float)(m64[2] * dx + m64[3] * dy);
    r.gb = (float)(m64[3] * dx + m64[4] * dy);
    r.p = eval_pair64(m64, B, px, py);
    return r;
}

// Transpose-reduce 16 values across a warp: afterwards lane L holds the warp sum of value
// index  ((L >> 1) & 15)  (lanes 2i and 2i+1 hold the same value).
__device__ __forceinline__ float warp_reduce16(float (&v)[16], int lane) {
#pragma unroll
    for (int half = 8, bit = 16; half >= 1; half >>= 1, bit >>= 1) {
        const bool upper = lane & bit;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = upper ? v[i] : v[i + half];
            const float keep = upper ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__device__ __forceinline__ float lg2_approx(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// One pixel per thread; a warp owns an 8x4 block.  The per-pair body is branch-free: a
// lane that does not take the pair (outside its last contributor, alpha < alpha_min) runs
// it with alpha = 0 and dL/dalpha = 0, which leaves its state (T, behind colour) exactly
// unchanged and all 11 partials exactly 0.
template <bool STATS>
__global__ void __launch_bounds__(BSR_BLOCK, 3) raster_bwd_kernel(RasterBwdArgs a) {
    constexpr int NW = BSR_BLOCK / 32;
    __shared__ __align__(16) Record s_recb[2][BSR_BLOCK];
    __shared__ uint32_t s_cidxb[2][BSR_BLOCK];
    __shared__ uint8_t s_list[NW][BSR_BLOCK];
    __shared__ int s_maxlast;
    const FrameView &f = a.f;
    const int tile = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int wx0 = tx * BSR_TILE + (warp & 1) * 8, wy0 = ty * BSR_TILE + (warp >> 1) * 4;
    const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
    const uint32_t *lists = a.lists ? a.lists : f.tvals[f.ctr->tile_plan[f.tile_passes] & 1u];
    const Record *rec = a.rec ? a.rec : f.rec;
    const uint2 range = (a.ranges ? a.ranges : f.tile_ranges)[tile];
    const int start = (int)range.x;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int direct_max = a.direct_max;

    int last = 0;
    float T = 1.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, gd = 0.f, B0 = a.bg[0], B1 = a.bg[1], B2 = a.bg[2], BD = 0.f;
    if (px < f.W && py < f.H) {
        const int64_t pix = (int64_t)py * f.W + px;
        const uint32_t packed = f.last[pix];
        last = (int)(packed & 0x1FFFFFFFu);
        if (last > 0) {
            T = f.t_final[pix];
            g0 = a.d_color[3 * pix];
            g1 = a.d_color[3 * pix + 1];
            g2 = a.d_color[3 * pix + 2];
            if (a.use_mask) {
                if (packed & (1u << 29)) g0 = 0.f;
                if (packed & (1u << 30)) g1 = 0.f;
                if (packed & (1u << 31)) g2 = 0.f;
            }
            if (a.d_depth) gd = a.d_depth[pix];
        }
    }
    int wlast = last;
    if (t == 0) s_maxlast = 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
    __syncthreads();
    if (lane == 0 && wlast) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int maxlast = s_maxlast;
    uint32_t pairs = 0;

    // batches [lo, hi) walked from the back; the next (earlier) batch is gathered with
    // cp.async while this one is processed
    auto prefetch = [&](int hi, int buf) {
        const int lo = max(0, hi - BSR_BLOCK);
        for (int q = t; q < hi - lo; q += BSR_BLOCK) {
            const uint32_t c = lists[start + lo + q];
            s_cidxb[buf][q] = c;
            const Record *src = rec + c;
            Record *dst = &s_recb[buf][q];
            cp_async16(&dst->a, &src->a);
            cp_async16(&dst->b, &src->b);
            cp_async16(&dst->c, &src->c);
            cp_async16(&dst->d, &src->d);
        }
        cp_async_commit();
    };
    if (maxlast > 0) prefetch(maxlast, 0);
    int buf = 0;
    for (int hi = maxlast; hi > 0; hi -= BSR_BLOCK, buf ^= 1) {
        const int lo = max(0, hi - BSR_BLOCK);
        const int nb = hi - lo;
        const bool more = lo > 0;
        __syncthreads();  // the buffer about to be refilled is no longer read
        if (more) prefetch(lo, buf ^ 1);
        if (more) cp_async_wait<1>(); else cp_async_wait<0>();
        __syncthreads();
        const Record *s_rec = s_recb[buf];
        const uint32_t *s_cidx = s_cidxb[buf];
        // ---- per-warp list: entries before the warp's furthest last contributor that
        //      reach its block (ascending; walked backwards)
        int nl = 0;
        if (wlast > lo) {
            for (int c0j = 0; c0j < nb; c0j += 32) {
                const int j = c0j + lane;
                bool hit = false;
                if (j < nb && lo + j < wlast) {
                    const Record &r = s_rec[j];
                    hit = STATS ? bbox_hits_rect(r.d, wx0, wx0 + 7, wy0, wy0 + 3)
                                : ellipse_hits_rect(r.a, r.b, r.c, r.d, wx0, wx0 + 7, wy0, wy0 + 3, a.alpha_min);
                }
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (hit) s_list[warp][nl + __popc(m & lt_mask)] = (uint8_t)j;
                nl += __popc(m);
            }
            __syncwarp();
        }
        for (int i = nl - 1; i >= 0; --i) {
            const int j = s_list[warp][i];
            const int e = lo + j;  // local entry index
            const int4 bd = s_rec[j].d;
            const float4 A = s_rec[j].a, Bq = s_rec[j].b, C = s_rec[j].c;
            if (STATS) pairs += (e < last && px >= bd.x && px <= bd.y && py >= bd.z && py <= bd.w);
            float ga, gb;  // (a dx + b dy, b dx + c dy): fp64 for unsafe primitives
            Pair p;
            if (C.w < 0.f) {  // fp32-unsafe primitive, uniform per entry
                const PairG u = unsafe_pair_bwd(f.rec64 + kRec64 * (int64_t)s_cidx[j], Bq, px, py);
                p = u.p;
                ga = u.ga;
                gb = u.gb;
            } else {
                p = eval_pair(A, Bq, px - bd.x, py - bd.z);
                ga = A.z * p.dx + A.w * p.dy;
                gb = A.w * p.dx + Bq.x * p.dy;
            }
            const bool took = e < last && p.alpha >= a.alpha_min;
            const unsigned tm = __ballot_sync(0xffffffffu, took);
            if (!tm) continue;
            const float alpha = took ? p.alpha : 0.f;
            const float one_m = 1.0f - alpha;     // alpha <= 0.999 (forward flags larger)
            T = took ? T * rcp_approx(one_m) : T;  // T_k
            const float w = alpha * T;
            float dalpha = T * (g0 * (C.x - B0) + g1 * (C.y - B1) + g2 * (C.z - B2) + gd * (Bq.w - BD));
            dalpha = took ? dalpha : 0.f;
            B0 = alpha * C.x + one_m * B0;
            B1 = alpha * C.y + one_m * B1;
            B2 = alpha * C.z + one_m * B2;
            BD = alpha * Bq.w + one_m * BD;
            // kernel derivative; a taken sample has alpha > 0, hence 1 - x > 0
            const float beta = Bq.z;
            const float om = fmaxf(p.om, 1e-30f);
            const float pw = beta == 4.0f ? om * om * om : p.k * rcp_approx(om);  // (1-x)^(beta-1)
            const float dk = dalpha * Bq.y;
            const float d_x = dk * fmaxf(-beta * pw, -kEdgeGradClamp);
            float v[16];
            v[0] = -2.0f * d_x * ga;
            v[1] = -2.0f * d_x * gb;
            v[2] = d_x * p.dx * p.dx;
            v[3] = 2.0f * d_x * p.dx * p.dy;
            v[4] = d_x * p.dy * p.dy;
            v[5] = dalpha * p.k;
            v[6] = dk * p.k * (0.69314718f * lg2_approx(om));
            v[7] = w * g0;
            v[8] = w * g1;
            v[9] = w * g2;
            v[10] = w * gd;
            float *dst = f.grad_acc + (int64_t)s_cidx[j] * kGradStride;
            if (__popc(tm) <= direct_max) {  // few contributors: direct atomics beat the reduction
                if (took) {
#pragma unroll
                    for (int q = 0; q < 11; ++q)
                        if (v[q] != 0.0f) atomicAdd(dst + q, v[q]);
                }
                continue;
            }
#pragma unroll
            for (int q = 11; q < 16; ++q) v[q] = 0.f;
            const float sum = warp_reduce16(v, lane);
            const int idx = (lane >> 1) & 15;
            if (!(lane & 1) && idx < 11 && sum != 0.0f) atomicAdd(dst + idx, sum);
        }
    }
    if (STATS) {
        unsigned long long p2 = pairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) p2 += __shfl_xor_sync(0xffffffffu, p2, o);
        if (lane == 0) atomicAdd(a.stats + 2, p2);
    }
}

int launch_raster_bwd(const FrameView &f, const float *d_color, bool use_mask, const float *d_depth,
                      const float bg[3], float alpha_min, const uint32_t *lists, const uint2 *ranges,
                      const Record *rec, unsigned long long *stats, cudaStream_t st) {
    if (f.n_tiles == 0) return BSR_OK;
    RasterBwdArgs a;
    a.f = f;
    a.d_color = d_color;
    a.use_mask = use_mask;
    a.d_depth = d_depth;
    a.bg[0] = bg[0];
    a.bg[1] = bg[1];
    a.bg[2] = bg[2];
    a.alpha_min = alpha_min;
    a.lists = lists;
    a.ranges = ranges;
    a.rec = rec;
    a.stats = stats;
    // warps with at most this many contributing lanes add their partials with direct
    // atomics instead of the 16-shuffle reduction (BSR_BWD_DIRECT overrides, for A/B)
    static const int direct_max = [] {
        const char *e = getenv("BSR_BWD_DIRECT");
        return e ? atoi(e) : 2;
    }();
    a.direct_max = direct_max;
    if (stats)
        raster_bwd_kernel<true><<<f.n_tiles, BSR_BLOCK, 0, st>>>(a);
    else
        raster_bwd_kernel<false><<<f.n_tiles, BSR_BLOCK, 0, st>>>(a);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
