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
// Per pair the 11 partials (geometry x5 in the whitened frame, d opacity, d beta, d rgb x3, d z)
// are reduced across the warp with a 16-shuffle transpose reduction and added with one
// warp-wide RED instruction per (warp, entry) into grad_acc[compact][12].
#include <stdlib.h>

#include <type_traits>

#include "raster.cuh"

#ifndef BSR_DENSE_X10
#define BSR_DENSE_X10 30  // dense mode when groups share entries; backward: from 3 groups per entry (measured: config 4 raster bwd 4.27 -> 4.22 ms from 2.5; worse above 3.5)
#endif

#ifndef BSR_NATURAL_TILE_ORDER
#define BSR_NATURAL_TILE_ORDER 0  // build knob for A/B runs: raster CTAs in tile-index order
#endif

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
    const uint32_t *emask;      // the forward's per-entry sub-block masks, or nullptr (computed here)
};

// fp64 pair evaluation for fp32-unsafe primitives; kept out of line so the common fp32
// path is not if-converted into predicated fp64 code.  With the record's fp64 factor
// (side64, positive-definite conic) the whitened coordinates u, w are formed in fp64 too.
__device__ __noinline__ Pair unsafe_pair_bwd(const double *m64, const double *s64, bool has_factor, float4 B,
                                             int px, int py) {
    Pair p = eval_pair64(m64, B, px, py);
    if (has_factor) {
        const double dx = (double)px - m64[0], dy = (double)py - m64[1];
        p.u = (float)(s64[0] * dx + s64[1] * dy);
        p.w = (float)(s64[2] * dy);
    }
    return p;
}

// xy-frame geometry partials in fp64 (frame.cuh add_geom64) of fp64-path records without a
// factor (conic not positive definite in fp64 -- practically never met), out of line like
// unsafe_pair_bwd.  Called by the whole warp when any lane took such a pair; the entry is
// uniform within each group of GL lanes, so the five partials are summed over the group in
// fp64 with shuffles and its first lane adds them.
template <int GL>
__device__ __noinline__ void unsafe_geom_bwd(double *side64, const double *rec64, DetAcc det, uint32_t c, float d_x,
                                             int px, int py, bool mine, unsigned gmask_any) {
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (mine) {
        const double *m64 = rec64 + kRec64 * (int64_t)c;
        const double dx = (double)px - m64[0], dy = (double)py - m64[1], dxx = (double)d_x;
        v[0] = -2.0 * dxx * (m64[2] * dx + m64[3] * dy);
        v[1] = -2.0 * dxx * (m64[3] * dx + m64[4] * dy);
        v[2] = dxx * dx * dx;
        v[3] = 2.0 * dxx * dx * dy;
        v[4] = dxx * dy * dy;
    }
#pragma unroll
    for (int o = GL / 2; o >= 1; o >>= 1)
#pragma unroll
        for (int q = 0; q < 5; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    const int lane = threadIdx.x & 31;
    if ((lane % GL) == 0 && ((gmask_any >> lane) & 1u)) {
        double *g = side64 + (int64_t)kSide64 * c;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            if (v[q] == 0.0) continue;
            if (det.mode)
                det_add(det, c, q, v[q]);
            else
                atomicAdd(g + q, v[q]);
        }
    }
}

// Transpose-reduce 16 values across the L lanes of a group (L = 32 / G): afterwards each
// lane holds group sums of NV = max(1, 32 / L / 2)... concretely
//   L = 32: lane k holds value (k >> 1)            (lanes 2i, 2i+1 equal), returned in r0
//   L = 16: lane k holds value k                    in r0
//   L =  8: lane k holds values 2k, 2k + 1          in r0, r1
template <int L>
__device__ __forceinline__ void group_reduce16(float (&v)[16], int lane, float &r0, float &r1) {
#pragma unroll
    for (int half = 8, bit = L / 2; half >= 1 && bit >= 1; half >>= 1, bit >>= 1) {
        const bool upper = lane & bit;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = upper ? v[i] : v[i + half];
            const float keep = upper ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
        }
    }
    if (L == 32) {
        r0 = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
        r1 = 0.f;
    } else {
        r0 = v[0];
        r1 = v[1];
    }
}
template <int L>
__device__ __forceinline__ int reduce_index(int k) {
    return L == 32 ? (k >> 1) : (L == 16 ? k : 2 * k);
}

__device__ __forceinline__ float lg2_approx(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// One pixel per thread; a warp owns an 8x4 block split into G sub-blocks whose lane groups
// walk their own entry lists (raster.cuh SubBlock).  The per-pair body is branch-free: a
// lane that does not take the pair (outside its last contributor, alpha < alpha_min, or
// its group's list exhausted) runs it with alpha = 0 and dL/dalpha = 0, which leaves its
// state (T, behind colour) exactly unchanged and all 11 partials exactly 0.
// MINB: resident CTAs per SM the register budget targets.  4 (64 registers, some spills)
// on frames of many tiles (config 4 raster bwd 4.42 -> 4.14 ms, config 3 0.771 -> 0.725 ms
// per view); 3 on small ones, where the full register file would keep the concurrent fp64
// replay's CTAs off the SMs until the raster's tail (config 1: 1.5-2% slower at 4)
constexpr int kBwdWideMinTiles = 4096;
// DET: 0 float atomics into grad_acc; 1 / 2 the deterministic bound / fixed-point passes
// (frame.cuh DetAcc) -- the same values, added through det_add.
template <bool STATS, int G, int DET, int MINB>
__global__ void __launch_bounds__(BSR_BLOCK, MINB) raster_bwd_kernel(RasterBwdArgs a) {
    pdl_wait();
    using SB = SubBlock<G>;
    using TG = TileGrid<G>;
    constexpr int L = SB::lanes;
    __shared__ __align__(16) Record s_recb[2][BSR_BLOCK];
    __shared__ uint32_t s_cidxb[2][BSR_BLOCK];
    __shared__ uint32_t s_col[BSR_BLOCK / 32][32];  // [chunk of 32 entries][tile sub-block]
    __shared__ int s_maxlast;
    const FrameView &f = a.f;
    // the frame's own tiles go heavy first (bin_scan's tile_order); the core seam's external
    // ranges keep the launch order
    const int tile = (a.ranges == nullptr && !BSR_NATURAL_TILE_ORDER) ? (int)a.f.tile_order[blockIdx.x] : (int)blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int wx0 = tx * BSR_TILE + (warp & 1) * 8, wy0 = ty * BSR_TILE + (warp >> 1) * 4;
    const int q = SB::group(lane);
    const int px = wx0 + SB::px(lane), py = wy0 + SB::py(lane);
    const uint32_t *lists = a.lists ? a.lists : f.lists;
    const Record *rec = a.rec ? a.rec : f.rec;
    const uint2 range = (a.ranges ? a.ranges : f.tile_ranges)[tile];
    const int start = (int)range.x;
    const int direct_max = a.direct_max;
    const int my_bit = TG::bit(warp, q);

    int last = 0;
    float T = 1.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, gd = 0.f, B0 = a.bg[0], B1 = a.bg[1], B2 = a.bg[2], BD = 0.f;
    if (px < f.W && py < f.H) {
        const int64_t pix = (int64_t)py * f.W + px;
        const uint32_t packed = f.last[pix];
        last = (int)(packed & 0x1FFFFFFFu);
        if (last > 0) {
            T = f.t_final[pix];
            if (T < 0.f) {  // flagged pixel: the entries before the flag point (replay.cu)
                T = -T;
                const float4 b = f.bwd_init[pix];
                B0 = b.x;
                B1 = b.y;
                B2 = b.z;
                BD = b.w;
            }
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
    // furthest last contributor of the group / warp / CTA
    int glast = last;
#pragma unroll
    for (int o = L / 2; o; o >>= 1) glast = max(glast, __shfl_xor_sync(0xffffffffu, glast, o));
    int wlast = glast;
#pragma unroll
    for (int o = 16; o >= L; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
    if (t == 0) s_maxlast = 0;
    __syncthreads();
    if (lane == 0 && wlast) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int maxlast = s_maxlast;
    uint32_t pairs = 0;

    // batches [lo, hi) walked from the back; the next (earlier) batch is gathered with
    // cp.async while this one is processed
    auto prefetch = [&](int hi, int buf) {
        const int lo = max(0, hi - BSR_BLOCK);
        for (int qq = t; qq < hi - lo; qq += BSR_BLOCK) {
            const uint32_t c = lists[start + lo + qq];
            s_cidxb[buf][qq] = c;
            const Record *src = rec + c;
            Record *dst = &s_recb[buf][qq];
            cp_async16(&dst->a, &src->a);
            cp_async16(&dst->b, &src->b);
            cp_async16(&dst->c, &src->c);
            cp_async16(&dst->d, &src->d);
        }
        cp_async_commit();
    };

    // one (pixel, entry) pair of the back-to-front replay (_raster.pyx:197-241) plus the
    // accumulation of its 11 partials; GL = lanes reduced together (32: the whole warp
    // walks one entry, L: every group its own)
    bool batch_nf = false;  // the current batch holds an fp64-path record without a factor
    const uint32_t srecb0 = (uint32_t)(__cvta_generic_to_shared(&s_recb[0][0]));
    const uint32_t scidxb0 = (uint32_t)(__cvta_generic_to_shared(&s_cidxb[0][0]));
    // rbase / cbase: shared-window addresses of the current batch's records / indices
    auto pair = [&](uint32_t rbase, uint32_t cbase, int lo, int j, bool act, auto gl_tag) {
        constexpr int GL = decltype(gl_tag)::value;
        const int e = lo + j;  // local entry index
        const uint32_t ra = rbase + (uint32_t)j * (uint32_t)sizeof(Record);
        const int4 bd = lds_i4(ra + 48);
        const float4 A = lds_f4(ra), Bq = lds_f4(ra + 16), C = lds_f4(ra + 32);
        const uint32_t cj = lds_u32(cbase + 4u * (uint32_t)j);
        if (STATS) pairs += (act && e < last && px >= bd.x && px <= bd.y && py >= bd.z && py <= bd.w);
        Pair p;
        bool geom64 = false;  // fp64-path record without a factor: xy-frame fp64 partials
        if (C.w < 0.f) {  // needle or fp64 primitive (uniform per entry)
            const uint32_t c = cj;
            const float4 N = f.needle[c];
            if (N.x == N.x) {  // needle: compensated fp32 (same bits as the forward)
                p = eval_needle(A, Bq, N, px - bd.x, py - bd.z);
            } else {
                p = unsafe_pair_bwd(f.rec64 + kRec64 * (int64_t)c, f.side64 + (int64_t)kSide64 * c, N.y != 0.f,
                                    Bq, px, py);
                geom64 = N.y == 0.f;
            }
        } else {
            p = eval_pair(A, Bq, px - bd.x, py - bd.z);
        }
        const bool took = act && e < last && p.alpha >= a.alpha_min;
        const unsigned tm = __ballot_sync(0xffffffffu, took);
        if (!tm) return;
        const float alpha = took ? p.alpha : 0.f;
        const float one_m = 1.0f - alpha;     // alpha <= 0.999 (forward flags larger)
        // T_k = T_{k+1} / (1 - alpha_k): rcp.approx plus one Newton step on the quotient, so the
        // recovered transmittance is (nearly) correctly rounded and unbiased -- the front
        // entries of a pixel recover T through every later entry, and a biased 1-ulp error per
        // step would add up linearly over thousands of entries at config 4
        const float rq = rcp_approx(one_m);
        const float q0 = __fmul_rn(T, rq);
        const float q1 = __fmaf_rn(__fmaf_rn(-q0, one_m, T), rq, q0);
        T = took ? q1 : T;  // T_k
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
        if (batch_nf) {  // rare: checked per batch so the common path has no extra vote
            const unsigned um = __ballot_sync(0xffffffffu, geom64 && took);
            if (um) {
                // group-leader lanes whose group has a contributing lane
                unsigned lead = 0u;
#pragma unroll
                for (int g = 0; g < 32 / GL; ++g) {
                    constexpr uint32_t gm = GL >= 32 ? 0xffffffffu : ((1u << (GL & 31)) - 1u);
                    if (um & (gm << ((g * GL) & 31))) lead |= 1u << ((g * GL) & 31);
                }
                unsafe_geom_bwd<GL>(f.side64, f.rec64, f.det, cj, d_x, px, py, geom64 && took, lead);
            }
        }
        // geometry partials in the record's whitened frame (frame.cuh grad_acc, factor L of
        // raster.cuh record_factor64): the components of sum d_x (u, w)(u, w)^T do not cancel
        // against each other the way the xy components of the conic gradient do for
        // elongated footprints (preprocess_bwd maps them back in fp64: d mean = -2 L (.),
        // d cov2d = -L (.) L^T)
        const float du = d_x * p.u, dw = d_x * p.w;
        v[0] = geom64 ? 0.f : du;
        v[1] = geom64 ? 0.f : dw;
        v[2] = geom64 ? 0.f : du * p.u;
        v[3] = geom64 ? 0.f : du * p.w;
        v[4] = geom64 ? 0.f : dw * p.w;
        v[5] = dalpha * p.k;
        v[6] = dk * p.k * (0.69314718f * lg2_approx(om));
        v[7] = w * g0;
        v[8] = w * g1;
        v[9] = w * g2;
        v[10] = w * gd;
        float *dst = f.grad_acc + (int64_t)cj * kGradStride;
        auto acc = [&](int k, float val) {
            if (DET == 0)
                atomicAdd(dst + k, val);
            else
                det_add(f.det, cj, k, (double)val);
        };
        // few contributors: direct atomics beat the reduction
        int most = __popc(tm);
        if (GL < 32) {
            most = 0;
            constexpr uint32_t gmask = GL >= 32 ? 0xffffffffu : ((1u << (GL & 31)) - 1u);
#pragma unroll
            for (int g = 0; g < 32 / GL; ++g) most = max(most, __popc(tm & (gmask << ((g * GL) & 31))));
        }
        if (most <= direct_max) {
            if (took) {
#pragma unroll
                for (int qq = 0; qq < 11; ++qq)
                    if (v[qq] != 0.0f) acc(qq, v[qq]);
            }
            return;
        }
#pragma unroll
        for (int qq = 11; qq < 16; ++qq) v[qq] = 0.f;
        float r0, r1;
        group_reduce16<GL>(v, lane, r0, r1);
        const int idx = reduce_index<GL>(lane % GL);
        if (GL == 32) {
            if (!(lane & 1) && idx < 11 && r0 != 0.0f) acc(idx, r0);
        } else {
            if (idx < 11 && r0 != 0.0f) acc(idx, r0);
            if (GL == 8 && idx + 1 < 11 && r1 != 0.0f) acc(idx + 1, r1);
        }
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
        const uint32_t rbase = srecb0 + (uint32_t)(buf * BSR_BLOCK) * (uint32_t)sizeof(Record);
        const uint32_t cbase = scidxb0 + 4u * (uint32_t)(buf * BSR_BLOCK);
        // ---- one thread per entry: which sub-blocks of the tile can it reach (bit columns
        //      per chunk of 32 entries, see raster_fwd.cu) -- the forward's masks when it kept
        //      them (the same entry_tile_mask; every entry before maxlast was reached by it)
        bool nf = false;
        {
            uint32_t m = 0;
            if (t < nb) {
                if (!STATS && a.emask) {
                    m = a.emask[start + lo + t];
                } else {
                    const Record &r = s_rec[t];
                    m = entry_tile_mask<G, STATS>(r.a, r.b, r.c, r.d, tx * BSR_TILE, ty * BSR_TILE, a.alpha_min);
                }
                if (s_rec[t].c.w < 0.f) {
                    const float4 N = f.needle[s_cidxb[buf][t]];
                    nf = N.x != N.x && N.y == 0.f;
                }
            }
            s_col[warp][lane] = warp_transpose32(m, lane);
        }
        batch_nf = __syncthreads_or(nf);
        if (wlast <= lo) continue;
        // entries [lo, lo + lim) precede the group's / warp's furthest last contributor
        const int glim = min(nb, glast - lo), wlim = min(nb, wlast - lo);
        bool dense = G == 1;
        if (G > 1) {
            int sum = 0, uni = 0;
            const int nch = (wlim + 31) >> 5;
            if (lane < nch) {
                uint32_t u = 0;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t cg = s_col[lane][TG::bit(warp, g)];
                    sum += __popc(cg);
                    u |= cg;
                }
                uni = __popc(u);
            }
#pragma unroll
            for (int o = 4; o; o >>= 1) {
                sum += __shfl_xor_sync(0xffffffffu, sum, o);
                uni += __shfl_xor_sync(0xffffffffu, uni, o);
            }
            // lanes 0..7 hold the totals; broadcast so the branch below is warp-uniform
            dense = __shfl_sync(0xffffffffu, 10 * sum >= BSR_DENSE_X10 * uni, 0);
        }
        // walk set bits from the highest entry below the limit down to entry 0
        auto lowbits = [](int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); };
        if (dense) {
            auto col = [&](int cc) {
                uint32_t u = 0;
#pragma unroll
                for (int g = 0; g < G; ++g) u |= s_col[cc][TG::bit(warp, g)];
                return u;
            };
            int c = (wlim - 1) >> 5;
            uint32_t bits = col(c) & lowbits(wlim - (c << 5));
            while (true) {
                while (!bits && c > 0) bits = col(--c);
                if (!bits) break;
                const int jb = 31 - __clz(bits);
                bits &= ~(1u << jb);
                pair(rbase, cbase, lo, (c << 5) + jb, true, std::integral_constant<int, 32>());
            }
        } else {
            int c = glim > 0 ? (glim - 1) >> 5 : -1;
            uint32_t bits = c >= 0 ? s_col[c][my_bit] & lowbits(glim - (c << 5)) : 0u;
            while (true) {
                while (!bits && c > 0) bits = s_col[--c][my_bit];
                if (!__any_sync(0xffffffffu, bits)) break;
                const bool act = bits != 0;
                const int jb = act ? 31 - __clz(bits) : 0;
                bits &= ~(1u << jb);
                pair(rbase, cbase, lo, act ? (c << 5) + jb : 0, act, std::integral_constant<int, L>());
            }
        }
    }
    if (STATS) {
        unsigned long long p2 = pairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) p2 += __shfl_xor_sync(0xffffffffu, p2, o);
        if (lane == 0) atomicAdd(a.stats + 2, p2);
    }
}

int raster_groups();

template <int G>
static int launch_bwd_g(const RasterBwdArgs &a, int tiles, bool stats, cudaStream_t st) {
    if (stats)
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<true, G, 0, 3>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (a.f.det.mode == 1 && tiles >= kBwdWideMinTiles)
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<false, G, 1, 4>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (a.f.det.mode == 1)
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<false, G, 1, 3>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (a.f.det.mode == 2 && tiles >= kBwdWideMinTiles)
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<false, G, 2, 4>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (a.f.det.mode == 2)
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<false, G, 2, 3>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (tiles >= kBwdWideMinTiles)
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<false, G, 0, 4>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else
        BSR_CUDA_TRY((pdl_launch(raster_bwd_kernel<false, G, 0, 3>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    return BSR_OK;
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
    a.emask = (lists == nullptr && f.entry_cap > 0) ? f.emask : nullptr;
    // warps with at most this many contributing lanes add their partials with direct
    // atomics instead of the 16-shuffle reduction (BSR_BWD_DIRECT overrides, for A/B)
    static const int direct_max = [] {
        const char *e = getenv("BSR_BWD_DIRECT");
        return e ? atoi(e) : 2;
    }();
    a.direct_max = direct_max;
    int rc = BSR_OK;
    switch (raster_groups()) {
        case 1: rc = launch_bwd_g<1>(a, f.n_tiles, stats != nullptr, st); break;
        case 2: rc = launch_bwd_g<2>(a, f.n_tiles, stats != nullptr, st); break;
        default: rc = launch_bwd_g<4>(a, f.n_tiles, stats != nullptr, st); break;
    }
    if (rc) return rc;
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
