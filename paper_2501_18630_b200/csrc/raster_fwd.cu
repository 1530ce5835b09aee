// K4 raster_fwd: per-16x16-tile front-to-back compositing (_raster.pyx:74-155).
//
// One CTA (256 threads) per tile, one pixel per thread; a warp owns an 8x4 pixel block,
// split into G sub-blocks of 32/G lanes that walk their own entry lists (raster.cuh).
// Tile-list records (64 B) are gathered into shared memory in batches of 256 with
// cp.async double buffering.  Per batch, every warp builds a compacted list of the entries
// whose ellipse actually reaches its 8x4 block (exact minimum of the conic over the block,
// one entry per lane, ballot-compacted), so the per-pixel loop only visits entries that
// can contribute to that warp.  Termination: the warp leaves its list once all its pixels
// reached T < t_stop, the CTA leaves the tile via __syncthreads_count ("composite, then
// stop", _raster.pyx:116-123).
//
// Exactness: the decisions alpha >= alpha_min and T < t_stop are taken in fp32
// only when a rigorous error bound certifies them; otherwise the pixel is handed to the
// fp64 replay (replay.cu) from that entry on.  Pixels with alpha > 0.999 (fp32 cannot
// carry 1 - alpha) are handed over too.
//
// Roofline: FP32 + XU pipes, per evaluated pair ~27 FP32 FLOP + 2 XU.
#include <stdlib.h>
#include <string.h>

#include "raster.cuh"

#ifndef BSR_DENSE_X10
#define BSR_DENSE_X10 40  // dense mode when groups share entries; forward: from 4 groups per entry (measured: config 4 raster fwd 2.76 -> 2.60 ms from 2.5)
#endif

#ifndef BSR_FWD_CTAS
#define BSR_FWD_CTAS 4  // resident CTAs per SM the register budget targets
#endif

#ifndef BSR_NATURAL_TILE_ORDER
#define BSR_NATURAL_TILE_ORDER 0  // build knob for A/B runs: raster CTAs in tile-index order
#endif

namespace bsr {

#ifdef BSR_FLAG_REASONS
// diagnostic build only: [alpha cutoff, alpha > 0.999, T stop, fp32 / needle / fp64 record]
__device__ unsigned long long g_flag_reasons[6];
extern "C" int bsr_debug_flag_reasons(unsigned long long *out, int reset) {
    cudaMemcpyFromSymbol(out, g_flag_reasons, sizeof(g_flag_reasons));
    if (reset) {
        unsigned long long z[6] = {0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_flag_reasons, z, sizeof(z));
    }
    return 0;
}
#endif

struct RasterFwdArgs {
    FrameView f;
    bsr_outputs out;
    float bg[3];
    float alpha_min, t_stop;
    // core seam: lists/ranges supplied externally instead of the frame's sorted buffers
    const uint32_t *lists;   // entry -> record index
    const uint2 *ranges;     // tile -> [start, end)
    const Record *rec;
    unsigned long long *stats;  // optional: [0] evaluated pairs, [1] contributions
    uint32_t *emask;            // optional: per-entry sub-block masks kept for the backward
};

// fp64 evaluation of an fp32-unsafe primitive, out of line so the common fp32 path is not
// if-converted into predicated fp64 code
// (only alpha and 1 - x leave the call: the fp32 error bounds are not used for it)
__device__ __noinline__ float2 unsafe_pair_fwd(const double *m64, float4 B, int px, int py) {
    const Pair p = eval_pair64(m64, B, px, py);
    return make_float2(p.alpha, p.om);
}

// COUNT: the deferred contributions pass (bsr_contributions): the same walk and decisions on
// the unchanged frame, counting only (no frame state, no outputs, no masks written)
template <bool STATS, bool CONTRIB, int G, bool COUNT = false>
__global__ void __launch_bounds__(BSR_BLOCK, BSR_FWD_CTAS) raster_fwd_kernel(RasterFwdArgs a) {
    pdl_wait();
    using SB = SubBlock<G>;
    using TG = TileGrid<G>;
    __shared__ __align__(16) Record s_rec[2][BSR_BLOCK];
    __shared__ uint32_t s_cidx[2][BSR_BLOCK];
    __shared__ uint32_t s_col[BSR_BLOCK / 32][32];  // [chunk of 32 entries][tile sub-block]
    __shared__ int s_cnt[BSR_BLOCK];
    __shared__ uint32_t s_mask[BSR_BLOCK];  // per-entry masks while several threads share an entry
    __shared__ int s_flag[BSR_BLOCK];  // entry where the pixel was handed to the fp64 replay (-1: none);
                                       // written once, kept out of the pair loop's registers
    const FrameView &f = a.f;
    // the frame's own tiles go heavy first (bin_scan's tile_order); the core seam's external
    // ranges keep the launch order
    const int tile = (a.ranges == nullptr && !BSR_NATURAL_TILE_ORDER) ? (int)a.f.tile_order[blockIdx.x] : (int)blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int wx0 = tx * BSR_TILE + (warp & 1) * 8, wy0 = ty * BSR_TILE + (warp >> 1) * 4;
    const int q = SB::group(lane);
    const int px = wx0 + SB::px(lane), py = wy0 + SB::py(lane);
    const bool inside = px < f.W && py < f.H;
    const uint32_t *lists = a.lists ? a.lists : f.lists;
    const Record *rec = a.rec ? a.rec : f.rec;
    const uint2 range = (a.ranges ? a.ranges : f.tile_ranges)[tile];
    const int start = (int)range.x, end = (int)range.y;
    constexpr bool want_contrib = CONTRIB;
    constexpr bool stats = STATS;
    const int my_bit = TG::bit(warp, q);

    float T = 1.0f, c0 = 0.f, c1 = 0.f, c2 = 0.f, dep = 0.f, errT = 0.f;  // errT: absolute bound on T's error
    int cnt = 0, last = 0;
    uint32_t pairs = 0;
    bool done = !inside;
    s_cnt[t] = 0;
    s_flag[t] = -1;

    auto prefetch = [&](int b0, int buf) {
        const int e = b0 + t;
        if (e < end) {
            const uint32_t c = lists[e];
            s_cidx[buf][t] = c;
            const Record *src = rec + c;
            Record *dst = &s_rec[buf][t];
            cp_async16(&dst->a, &src->a);
            cp_async16(&dst->b, &src->b);
            cp_async16(&dst->c, &src->c);
            cp_async16(&dst->d, &src->d);
        }
        cp_async_commit();
    };

    const uint32_t srec0 = (uint32_t)(__cvta_generic_to_shared(&s_rec[0][0]));
    const uint32_t scidx0 = (uint32_t)(__cvta_generic_to_shared(&s_cidx[0][0]));
    // one (pixel, entry) pair of the front-to-back composite (_raster.pyx:101-123)
    auto pair = [&](int b0, int buf, int j) -> bool {
        bool took = false;
        const uint32_t ra = srec0 + (uint32_t)(buf * BSR_BLOCK + j) * (uint32_t)sizeof(Record);
        const int4 bd = lds_i4(ra + 48);
        if (stats) pairs += (px >= bd.x && px <= bd.y && py >= bd.z && py <= bd.w);
        const float4 A = lds_f4(ra), B = lds_f4(ra + 16), C = lds_f4(ra + 32);
        const uint32_t cj = lds_u32(scidx0 + 4u * (uint32_t)(buf * BSR_BLOCK + j));
        const bool unsafe = C.w < 0.f;  // needle or fp64 record (uniform per entry)
        const float Q = fabsf(C.w);
        bool fp64 = false;
        Pair p;
        if (unsafe) {
            const float4 N = f.needle[cj];
            if (N.x == N.x) {  // needle: compensated fp32
                p = eval_needle(A, B, N, px - bd.x, py - bd.z);
            } else {
                fp64 = true;
                const float2 u = unsafe_pair_fwd(f.rec64 + kRec64 * (int64_t)cj, B, px, py);
                p.alpha = u.x;
                p.om = u.y;
            }
        } else {
            p = eval_pair(A, B, px - bd.x, py - bd.z);
        }
        // most evaluated pairs are well below the cutoff: one compare leaves them (the
        // tests below cannot pass for alpha below ~0.9 alpha_min; no extra live register)
        if (!(p.alpha * 1.1111111f >= a.alpha_min)) return false;
        bool ambiguous = false;
        // rare path: alpha within 5% of the cutoff -> certify with the error bound
        if (fabsf(p.alpha - a.alpha_min) < 0.05f * a.alpha_min) {
            const float rel = fp64 ? 8.0f * kEps
                                   : (unsafe ? Q * rcp_approx(fmaxf(p.om, 1e-30f)) * 1.01f
                                             : alpha_rel_err_pixel(A, B, p));
            ambiguous = fabsf(p.alpha - a.alpha_min) <= 2.0f * rel * p.alpha + 4.0f * kEps * a.alpha_min;
        }
        if (!ambiguous && p.alpha >= a.alpha_min) {
            const float one_m = __fsub_rn(1.0f, p.alpha);
            const float Tn = __fmul_rn(T, one_m);
            // absolute error bound of T (T_c = T + dT, alpha_c = alpha + da):
            //   dTn <= (1 - alpha) dT + T |da| + 2.5 eps Tn,
            // |da| <= alpha Q / om (record_err_word); for beta = 4, alpha = o om^4, so
            // alpha / om = o om^3 needs no reciprocal
            const float da = fp64 ? 8.0f * kEps * p.alpha
                                  : (B.z == 4.0f ? Q * (B.y * (p.om * p.om * p.om))
                                                 : p.alpha * Q * rcp_approx(fmaxf(p.om, 1e-30f)));
            const float errTn = one_m * errT + 1.01f * T * da + 2.5f * kEps * Tn;
            if (p.alpha > 0.999f || fabsf(Tn - a.t_stop) <= 2.0f * errTn + 4.0f * kEps * a.t_stop) {
                ambiguous = true;
            } else {
                const float w = __fmul_rn(p.alpha, T);
                c0 = __fmaf_rn(w, C.x, c0);
                c1 = __fmaf_rn(w, C.y, c1);
                c2 = __fmaf_rn(w, C.z, c2);
                dep = __fmaf_rn(w, B.w, dep);
                T = Tn;
                errT = errTn;
                ++cnt;
                last = b0 + j - start + 1;
                took = true;
                if (T < a.t_stop) done = true;
            }
        }
        if (ambiguous) {
#ifdef BSR_FLAG_REASONS
            atomicAdd(&g_flag_reasons[p.alpha > 0.999f ? 1 : (p.alpha >= a.alpha_min && fabsf(p.alpha - a.alpha_min) >= 0.05f * a.alpha_min) ? 2 : 0], 1ull);
            atomicAdd(&g_flag_reasons[3 + (fp64 ? 2 : unsafe ? 1 : 0)], 1ull);
#endif
            s_flag[t] = b0 + j - start;
            done = true;
        }
        return took;
    };

    if (start < end) prefetch(start, 0);
    int buf = 0;
    int reached = start;  // emask written for [start, reached)
    for (int b0 = start; b0 < end; b0 += BSR_BLOCK, buf ^= 1) {
        const bool more = b0 + BSR_BLOCK < end;
        if (more) prefetch(b0 + BSR_BLOCK, buf ^ 1);
        if (more) cp_async_wait<1>(); else cp_async_wait<0>();
        if (__syncthreads_count(done) == BSR_BLOCK) break;
        const int nb = min(BSR_BLOCK, end - b0);
        const int nch = (nb + 31) >> 5;
        // ---- one thread per entry: which sub-blocks of the tile can it reach; transposed
        //      per chunk of 32 entries into one bit column per sub-block
        batch_masks<G, stats>(s_rec[buf], nb, tx * BSR_TILE, ty * BSR_TILE, a.alpha_min, s_mask, s_col,
                              a.emask ? a.emask + b0 : nullptr);
        reached = b0 + nb;
        __syncthreads();
        // ---- this warp's groups: open (some pixel not finished) and how much their entry
        //      sets overlap; groups that mostly share entries walk the union together
        //      ("dense": one entry per warp-iteration), otherwise each group walks its own
        const unsigned done_b = __ballot_sync(0xffffffffu, done);
        const bool my_open = (done_b & SB::mask(q)) != SB::mask(q);
        bool dense = G == 1;
        if (G > 1) {
            int sum = 0, uni = 0;
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
        if (dense) {
            int c = 0;
            auto col = [&](int cc) {
                uint32_t u = 0;
#pragma unroll
                for (int g = 0; g < G; ++g) u |= s_col[cc][TG::bit(warp, g)];
                return u;
            };
            uint32_t bits = col(0);
            while (true) {
                while (!bits && c + 1 < nch) bits = col(++c);
                if (!bits || __all_sync(0xffffffffu, done)) break;
                const int j = (c << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                const bool took = !done && pair(b0, buf, j);
                if (want_contrib) {
                    const unsigned bl = __ballot_sync(0xffffffffu, took);
                    if (bl && lane == 0) atomicAdd(&s_cnt[j], __popc(bl));
                }
            }
        } else {
            int c = my_open ? 0 : nch;
            uint32_t bits = my_open ? s_col[0][my_bit] : 0u;
            while (true) {
                while (!bits && c + 1 < nch) bits = s_col[++c][my_bit];
                if (__all_sync(0xffffffffu, done || !bits)) break;
                const bool act = bits != 0;
                const int j = act ? (c << 5) + __ffs(bits) - 1 : 0;
                bits &= bits - 1;
                const bool took = act && !done && pair(b0, buf, j);
                if (want_contrib) {
                    const unsigned gb = __ballot_sync(0xffffffffu, took) & SB::mask(q);
                    if (gb && lane == q * SB::lanes) atomicAdd(&s_cnt[j], __popc(gb));
                }
            }
        }
        __syncthreads();
        if (want_contrib && t < nb && s_cnt[t]) {
            atomicAdd(a.out.contributions + s_cidx[buf][t], s_cnt[t]);
            s_cnt[t] = 0;
        }
    }
    cp_async_wait<0>();
    if (COUNT) return;
    if (a.emask && t == 0) f.mask_end[tile] = (uint32_t)reached;  // the replay's entry pre-test
    if (stats) {
        unsigned long long p2 = pairs, c2s = (unsigned)cnt;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            p2 += __shfl_xor_sync(0xffffffffu, p2, o);
            c2s += __shfl_xor_sync(0xffffffffu, c2s, o);
        }
        if (lane == 0) {
            atomicAdd(a.stats, p2);
            atomicAdd(a.stats + 1, c2s);
        }
    }
    if (!inside) return;
    const int64_t pix = (int64_t)py * f.W + px;
    const int flag_at = s_flag[t];
    if (flag_at >= 0) {
        const uint32_t slot = atomicAdd(&f.ctr->flagged, 1u);
        f.flags[slot] = make_uint2((uint32_t)pix, (uint32_t)flag_at);
        // the certified entries before the flag stay with the fp32 backward: it walks
        // [0, last) from this T (sign-marked; the replay adds the clamp bits and the state
        // behind the flag point, bwd_init); every per-pixel output is written by the replay
        f.t_final[pix] = -T;
        f.last[pix] = (uint32_t)last;
        return;
    }
    const float r0 = __fmaf_rn(a.bg[0], T, c0), r1 = __fmaf_rn(a.bg[1], T, c1),
                r2 = __fmaf_rn(a.bg[2], T, c2);
    f.t_final[pix] = T;
    // low 29 bits: local end index of the last contributor; bits 29..31: raw < 0 per
    // channel (clamp chain of the backward, rasterizer.py:253)
    f.last[pix] = (uint32_t)last | (!(r0 >= 0.f) ? 1u << 29 : 0u) | (!(r1 >= 0.f) ? 1u << 30 : 0u) |
                  (!(r2 >= 0.f) ? 1u << 31 : 0u);
    if (a.out.raw) {
        a.out.raw[3 * pix] = r0;
        a.out.raw[3 * pix + 1] = r1;
        a.out.raw[3 * pix + 2] = r2;
    }
    if (a.out.color) {
        a.out.color[3 * pix] = fmaxf(r0, 0.f);
        a.out.color[3 * pix + 1] = fmaxf(r1, 0.f);
        a.out.color[3 * pix + 2] = fmaxf(r2, 0.f);
    }
    if (a.out.alpha) a.out.alpha[pix] = 1.0f - T;
    if (a.out.transmittance) a.out.transmittance[pix] = T;
    if (a.out.depth) a.out.depth[pix] = dep;
    if (a.out.pixel_count) a.out.pixel_count[pix] = cnt;
}

// sub-warp groups per warp (1: 8x4, 2: 4x4, 4: 4x2 pixel sub-blocks); BSR_RASTER_G
// overrides for A/B measurements
int raster_groups() {
    static const int g = [] {
        const char *e = getenv("BSR_RASTER_G");
        const int v = e ? atoi(e) : 4;
        return (v == 1 || v == 2 || v == 4) ? v : 4;
    }();
    return g;
}

template <int G>
static int launch_fwd_g(const RasterFwdArgs &a, int tiles, bool stats, bool contrib, cudaStream_t st) {
    if (stats && contrib)
        BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<true, true, G>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (stats)
        BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<true, false, G>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else if (contrib)
        BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<false, true, G>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    else
        BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<false, false, G>, dim3(tiles), dim3(BSR_BLOCK), 0, st, a)));
    return BSR_OK;
}

// the deferred contributions pass: the frame's own lists, masks recomputed (not stored)
int launch_raster_count(const FrameView &f, int32_t *contributions, const float bg[3], float alpha_min,
                        float t_stop, cudaStream_t st) {
    if (f.n_tiles == 0) return BSR_OK;
    RasterFwdArgs a;
    memset(&a, 0, sizeof(a));
    a.f = f;
    a.out.contributions = contributions;
    a.bg[0] = bg[0];
    a.bg[1] = bg[1];
    a.bg[2] = bg[2];
    a.alpha_min = alpha_min;
    a.t_stop = t_stop;
    a.emask = nullptr;
    switch (raster_groups()) {
        case 1: BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<false, true, 1, true>, dim3(f.n_tiles), dim3(BSR_BLOCK), 0, st, a))); break;
        case 2: BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<false, true, 2, true>, dim3(f.n_tiles), dim3(BSR_BLOCK), 0, st, a))); break;
        default: BSR_CUDA_TRY((pdl_launch(raster_fwd_kernel<false, true, 4, true>, dim3(f.n_tiles), dim3(BSR_BLOCK), 0, st, a))); break;
    }
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

int launch_raster_fwd(const FrameView &f, const bsr_outputs &out, const float bg[3], float alpha_min,
                      float t_stop, const uint32_t *lists, const uint2 *ranges, const Record *rec,
                      unsigned long long *stats, cudaStream_t st) {
    if (f.n_tiles == 0) return BSR_OK;
    RasterFwdArgs a;
    a.f = f;
    a.out = out;
    a.bg[0] = bg[0];
    a.bg[1] = bg[1];
    a.bg[2] = bg[2];
    a.alpha_min = alpha_min;
    a.t_stop = t_stop;
    a.lists = lists;
    a.ranges = ranges;
    a.rec = rec;
    a.stats = stats;
    // the frame's own lists (not the core seam's external ones): keep the entry masks
    a.emask = (lists == nullptr && f.entry_cap > 0) ? f.emask : nullptr;
    const bool contrib = out.contributions != nullptr, st_on = stats != nullptr;
    int rc = BSR_OK;
    switch (raster_groups()) {
        case 1: rc = launch_fwd_g<1>(a, f.n_tiles, st_on, contrib, st); break;
        case 2: rc = launch_fwd_g<2>(a, f.n_tiles, st_on, contrib, st); break;
        default: rc = launch_fwd_g<4>(a, f.n_tiles, st_on, contrib, st); break;
    }
    if (rc) return rc;
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
