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

__global__ void __launch_bounds__(BSR_BLOCK, 3) raster_bwd_kernel(RasterBwdArgs a) {
    __shared__ __align__(16) Record s_rec[BSR_BLOCK];
    __shared__ uint32_t s_cidx[BSR_BLOCK];
    __shared__ uint8_t s_list[BSR_BLOCK / 32][BSR_BLOCK];
    __shared__ int s_maxlast;
    const FrameView &f = a.f;
    const int tile = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int wx0 = tx * BSR_TILE + (warp & 1) * 8, wy0 = ty * BSR_TILE + (warp >> 1) * 4;
    const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
    const bool inside = px < f.W && py < f.H;
    const uint32_t *lists = a.lists ? a.lists : f.tvals[f.ctr->tile_plan[f.tile_passes] & 1u];
    const Record *rec = a.rec ? a.rec : f.rec;
    const uint2 range = (a.ranges ? a.ranges : f.tile_ranges)[tile];
    const int start = (int)range.x;
    const bool stats = a.stats != nullptr;
    const uint32_t lt_mask = (1u << lane) - 1u;

    const int64_t pix = (int64_t)py * f.W + px;
    int last = 0;
    float T = 1.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, gd = 0.f;
    if (inside) {
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
    if (t == 0) s_maxlast = 0;
    int wlast = last;
#pragma unroll
    for (int o = 16; o; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
    __syncthreads();
    if (lane == 0 && wlast) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int maxlast = s_maxlast;
    float B0 = a.bg[0], B1 = a.bg[1], B2 = a.bg[2], BD = 0.f;
    uint32_t pairs = 0;

    for (int hi = maxlast; hi > 0; hi -= BSR_BLOCK) {
        const int lo = max(0, hi - BSR_BLOCK);
        const int nb = hi - lo;
        __syncthreads();
        if (t < nb) {
            const uint32_t c = lists[start + lo + t];
            s_cidx[t] = c;
            s_rec[t] = rec[c];
        }
        __syncthreads();
        // ---- per-warp list: entries before the warp's furthest last contributor that
        //      reach its 8x4 block (ascending; walked backwards)
        int nl = 0;
        if (wlast > lo) {
            for (int c0j = 0; c0j < nb; c0j += 32) {
                const int j = c0j + lane;
                bool hit = false;
                if (j < nb && lo + j < wlast) {
                    const Record &r = s_rec[j];
                    hit = stats ? bbox_hits_rect(r.d, wx0, wx0 + 7, wy0, wy0 + 3)
                                : ellipse_hits_rect(r.a, r.b, r.c, r.d, wx0, wx0 + 7, wy0, wy0 + 3);
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
            const bool act = e < last;
            float v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = 0.f;
            bool took = false;
            if (act) {
                const int4 bd = s_rec[j].d;
                if (stats) pairs += (px >= bd.x && px <= bd.y && py >= bd.z && py <= bd.w);
                const float4 A = s_rec[j].a, Bq = s_rec[j].b, C = s_rec[j].c;
                const double *m64 = C.w < 0.f ? f.rec64 + kRec64 * (int64_t)s_cidx[j] : nullptr;
                const Pair p = m64 ? eval_pair64(m64, Bq, px, py) : eval_pair(A, Bq, px - bd.x, py - bd.z);
                if (p.alpha >= a.alpha_min) {
                    took = true;
                    const float one_m = 1.0f - p.alpha;
                    T = T / one_m;  // T_k
                    const float w = p.alpha * T;
                    const float dalpha =
                        T * (g0 * (C.x - B0) + g1 * (C.y - B1) + g2 * (C.z - B2) + gd * (Bq.w - BD));
                    B0 = p.alpha * C.x + one_m * B0;
                    B1 = p.alpha * C.y + one_m * B1;
                    B2 = p.alpha * C.z + one_m * B2;
                    BD = p.alpha * Bq.w + one_m * BD;
                    v[7] = w * g0;
                    v[8] = w * g1;
                    v[9] = w * g2;
                    v[10] = w * gd;
                    v[5] = dalpha * p.k;
                    const float dk = dalpha * Bq.y;
                    if (p.x < 1.0f) {
                        const float beta = Bq.z;
                        // (1-x)^(beta-1) = k / (1-x); ln(1-x) via the XU pipe
                        const float pw = beta == 4.0f ? p.om * p.om * p.om : p.k / p.om;
                        v[6] = dk * p.k * __logf(p.om);
                        float dkdx = -beta * pw;
                        if (dkdx < -kEdgeGradClamp) dkdx = -kEdgeGradClamp;
                        const float d_x = dk * dkdx;
                        float ga, gb;  // (a dx + b dy, b dx + c dy): fp64 for unsafe primitives
                        if (m64) {
                            const double dx = (double)px - m64[0], dy = (double)py - m64[1];
                            ga = (float)(m64[2] * dx + m64[3] * dy);
                            gb = (float)(m64[3] * dx + m64[4] * dy);
                        } else {
                            ga = A.z * p.dx + A.w * p.dy;
                            gb = A.w * p.dx + Bq.x * p.dy;
                        }
                        v[0] = -d_x * 2.0f * ga;
                        v[1] = -d_x * 2.0f * gb;
                        v[2] = d_x * p.dx * p.dx;
                        v[3] = d_x * 2.0f * p.dx * p.dy;
                        v[4] = d_x * p.dy * p.dy;
                    }
                }
            }
            if (!__any_sync(0xffffffffu, took)) continue;
            const float sum = warp_reduce16(v, lane);
            const int idx = (lane >> 1) & 15;
            if (!(lane & 1) && idx < 11 && sum != 0.0f)
                atomicAdd(f.grad_acc + (int64_t)s_cidx[j] * kGradStride + idx, sum);
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
    raster_bwd_kernel<<<f.n_tiles, BSR_BLOCK, 0, st>>>(a);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

}  // namespace bsr
