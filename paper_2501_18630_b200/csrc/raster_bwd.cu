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
};

// fp64 pair evaluation + the two conic-gradient terms for fp32-unsafe primitives; kept
// out of line so the common fp32 path is not if-converted into predicated fp64 code.
__device__ __noinline__ Pair unsafe_pair_bwd(const double *m64, float4 B, int px, int py, float *ga, float *gb) {
    const double dx = (double)px - m64[0], dy = (double)py - m64[1];
    *ga = (float)(m64[2] * dx + m64[3] * dy);
    *gb = (float)(m64[3] * dx + m64[4] * dy);
    return eval_pair64(m64, B, px, py);
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

// PIX pixels per thread (stacked vertically 4 rows apart): a warp owns an 8 x 4*PIX block,
// so the per-(warp, entry) costs -- record loads, list walk, the reduction, the atomics --
// are shared by 32*PIX pixels.
template <int PIX, int MINB, bool STATS>
__global__ void __launch_bounds__(BSR_BLOCK / PIX, MINB) raster_bwd_kernel(RasterBwdArgs a) {
    constexpr int NT = BSR_BLOCK / PIX, NW = NT / 32, WH = 4 * PIX;
    __shared__ __align__(16) Record s_recb[2][BSR_BLOCK];
    __shared__ uint32_t s_cidxb[2][BSR_BLOCK];
    __shared__ uint8_t s_list[NW][BSR_BLOCK];
    __shared__ int s_maxlast;
    const FrameView &f = a.f;
    const int tile = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int wx0 = tx * BSR_TILE + (warp & 1) * 8, wy0 = ty * BSR_TILE + (warp >> 1) * WH;
    const int px = wx0 + (lane & 7);
    const uint32_t *lists = a.lists ? a.lists : f.tvals[f.ctr->tile_plan[f.tile_passes] & 1u];
    const Record *rec = a.rec ? a.rec : f.rec;
    const uint2 range = (a.ranges ? a.ranges : f.tile_ranges)[tile];
    const int start = (int)range.x;
    constexpr bool stats = STATS;
    const uint32_t lt_mask = (1u << lane) - 1u;

    int py[PIX], last[PIX];
    float T[PIX], g0[PIX], g1[PIX], g2[PIX], gd[PIX], B0[PIX], B1[PIX], B2[PIX], BD[PIX];
    int wlast = 0;
#pragma unroll
    for (int q = 0; q < PIX; ++q) {
        py[q] = wy0 + (lane >> 3) + 4 * q;
        last[q] = 0;
        T[q] = 1.f;
        g0[q] = g1[q] = g2[q] = gd[q] = 0.f;
        B0[q] = a.bg[0];
        B1[q] = a.bg[1];
        B2[q] = a.bg[2];
        BD[q] = 0.f;
        if (px < f.W && py[q] < f.H) {
            const int64_t pix = (int64_t)py[q] * f.W + px;
            const uint32_t packed = f.last[pix];
            last[q] = (int)(packed & 0x1FFFFFFFu);
            if (last[q] > 0) {
                T[q] = f.t_final[pix];
                g0[q] = a.d_color[3 * pix];
                g1[q] = a.d_color[3 * pix + 1];
                g2[q] = a.d_color[3 * pix + 2];
                if (a.use_mask) {
                    if (packed & (1u << 29)) g0[q] = 0.f;
                    if (packed & (1u << 30)) g1[q] = 0.f;
                    if (packed & (1u << 31)) g2[q] = 0.f;
                }
                if (a.d_depth) gd[q] = a.d_depth[pix];
            }
        }
        wlast = max(wlast, last[q]);
    }
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
        for (int q = t; q < hi - lo; q += NT) {
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
                    hit = stats ? bbox_hits_rect(r.d, wx0, wx0 + 7, wy0, wy0 + WH - 1)
                                : ellipse_hits_rect(r.a, r.b, r.c, r.d, wx0, wx0 + 7, wy0, wy0 + WH - 1, a.alpha_min);
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
            const bool unsafe = C.w < 0.f;  // uniform per entry
            float v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = 0.f;
            bool took = false;
#pragma unroll
            for (int q = 0; q < PIX; ++q) {
                if (e >= last[q]) continue;
                if (stats) pairs += (px >= bd.x && px <= bd.y && py[q] >= bd.z && py[q] <= bd.w);
                float ga, gb;  // (a dx + b dy, b dx + c dy): fp64 for unsafe primitives
                Pair p;
                if (unsafe) {
                    p = unsafe_pair_bwd(f.rec64 + kRec64 * (int64_t)s_cidx[j], Bq, px, py[q], &ga, &gb);
                } else {
                    p = eval_pair(A, Bq, px - bd.x, py[q] - bd.z);
                    ga = A.z * p.dx + A.w * p.dy;
                    gb = A.w * p.dx + Bq.x * p.dy;
                }
                if (!(p.alpha >= a.alpha_min)) continue;
                took = true;
                const float one_m = 1.0f - p.alpha;
                T[q] = __fdividef(T[q], one_m);  // T_k
                const float w = p.alpha * T[q];
                const float dalpha = T[q] * (g0[q] * (C.x - B0[q]) + g1[q] * (C.y - B1[q]) +
                                             g2[q] * (C.z - B2[q]) + gd[q] * (Bq.w - BD[q]));
                B0[q] = p.alpha * C.x + one_m * B0[q];
                B1[q] = p.alpha * C.y + one_m * B1[q];
                B2[q] = p.alpha * C.z + one_m * B2[q];
                BD[q] = p.alpha * Bq.w + one_m * BD[q];
                v[7] += w * g0[q];
                v[8] += w * g1[q];
                v[9] += w * g2[q];
                v[10] += w * gd[q];
                v[5] += dalpha * p.k;
                const float dk = dalpha * Bq.y;
                if (p.x < 1.0f) {
                    const float beta = Bq.z;
                    // (1-x)^(beta-1) = k / (1-x); ln(1-x) via the XU pipe
                    const float pw = beta == 4.0f ? p.om * p.om * p.om : p.k / p.om;
                    v[6] += dk * p.k * __logf(p.om);
                    float dkdx = -beta * pw;
                    if (dkdx < -kEdgeGradClamp) dkdx = -kEdgeGradClamp;
                    const float d_x = dk * dkdx;
                    v[0] += -d_x * 2.0f * ga;
                    v[1] += -d_x * 2.0f * gb;
                    v[2] += d_x * p.dx * p.dx;
                    v[3] += d_x * 2.0f * p.dx * p.dy;
                    v[4] += d_x * p.dy * p.dy;
                }
            }
            const unsigned tm = __ballot_sync(0xffffffffu, took);
            if (!tm) continue;
            float *dst = f.grad_acc + (int64_t)s_cidx[j] * kGradStride;
            if (__popc(tm) <= 2) {  // few contributors: direct atomics beat a 62-op reduction
                if (took) {
#pragma unroll
                    for (int q = 0; q < 11; ++q)
                        if (v[q] != 0.0f) atomicAdd(dst + q, v[q]);
                }
                continue;
            }
            const float sum = warp_reduce16(v, lane);
            const int idx = (lane >> 1) & 15;
            if (!(lane & 1) && idx < 11 && sum != 0.0f) atomicAdd(dst + idx, sum);
        }
    }
    if (stats) {
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
    // variant selection for A/B measurements (default: one pixel per thread, 3 CTAs/SM)
    static const int variant = [] {
        const char *e = getenv("BSR_BWD_VARIANT");
        return e ? atoi(e) : 0;
    }();
    if (stats)
        raster_bwd_kernel<1, 3, true><<<f.n_tiles, BSR_BLOCK, 0, st>>>(a);
    else if (variant == 1)
        raster_bwd_kernel<1, 4, false><<<f.n_tiles, BSR_BLOCK, 0, st>>>(a);
    else if (variant == 2)
        raster_bwd_kernel<2, 5, false><<<f.n_tiles, BSR_BLOCK / 2, 0, st>>>(a);
    else
        raster_bwd_kernel<1, 3, false><<<f.n_tiles, BSR_BLOCK, 0, st>>>(a);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
