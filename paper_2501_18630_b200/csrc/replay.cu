// fp64 replay of the pixels the fp32 raster could not certify.
//
// Flagged pixels are re-walked with the reference's fp64 arithmetic (_raster.pyx:101-127
// forward, :191-241 backward; this file is compiled with -fmad=false like pkg/setup.py's
// -ffp-contract=off).  Primitive values come from a Provider: the full pipeline reads the
// fp64 geometry preprocess wrote (project.cuh), the core seam the caller's fp64 arrays.
// Only list entries whose forward sub-block mask reaches the pixel are evaluated (the
// mask pre-test, MaskTest).
//
// Forward (one CTA per pixel): the whole list in fp64, writes every per-pixel output and
// counts contributions of entries at or after the entry where fp32 stopped (entries before
// it were certified and counted by the fp32 kernel); it also records the split point.
// Backward: the certified entries before the split point go through the fp32 raster
// backward (raster_fwd.cu marks the pixel, store_split leaves its starting state); the
// replay adds the gradients of the entries from the split point on (one CTA per pixel on
// small frames, one warp per pixel on large ones).
#include <stdlib.h>

#include "frame.cuh"
#include "appearance.cuh"
#include "project.cuh"
#include "raster.cuh"

namespace bsr {

struct Entry64 {
    double mx, my, ca, cb, cc, o, beta, r, g, b, z;
    int src;
};

// Full pipeline: recompute from the scene parameters (bit-identical to preprocess).
template <int K>
struct SceneProvider {
    bsr_scene sc;
    KCam cam;
    const Record *rec;
    const double *rec64;
    // fp64 geometry written by preprocess (project64, the same code and bits as the
    // reference restatement); the colour is the record's (fp32-evaluated, as on every
    // certified pixel: colour never enters a decision, only the blended value)
    __device__ __forceinline__ bool get(uint32_t c, int px, int py, Entry64 &e) const {
        const Record &r = rec[c];
        const int4 bd = r.d;
        const float4 col = r.c;
        if (px < bd.x || px > bd.y || py < bd.z || py > bd.w) return false;
        const double4 *d = reinterpret_cast<const double4 *>(rec64 + kRec64 * (int64_t)c);
        const double4 d0 = d[0], d1 = d[1];
        e.mx = d0.x;
        e.my = d0.y;
        e.ca = d0.z;
        e.cb = d0.w;
        e.cc = d1.x;
        e.o = d1.y;
        e.beta = d1.z;
        e.z = d1.w;
        e.r = col.x;
        e.g = col.y;
        e.b = col.z;
        e.src = (int)c;
        return true;
    }
    __device__ __forceinline__ void color(Entry64 &) const {}
};

// Core seam: the caller's depth-sorted fp64 arrays (_raster.pyx:130-134 inputs).
struct ArrayProvider {
    const double *means, *conics, *opac, *betas, *colors;
    const int32_t *bounds;
    __device__ __forceinline__ bool get(uint32_t c, int px, int py, Entry64 &e) const {
        const int32_t *bd = bounds + 4 * (int64_t)c;
        if (px < bd[0] || px > bd[1] || py < bd[2] || py > bd[3]) return false;
        e.mx = means[2 * c];
        e.my = means[2 * c + 1];
        e.ca = conics[3 * c];
        e.cb = conics[3 * c + 1];
        e.cc = conics[3 * c + 2];
        e.o = opac[c];
        e.beta = betas[c];
        e.z = 0.0;
        e.src = (int)c;
        return true;
    }
    __device__ __forceinline__ void color(Entry64 &e) const {
        const int64_t c = e.src;
        e.r = colors[3 * c];
        e.g = colors[3 * c + 1];
        e.b = colors[3 * c + 2];
    }
};

struct ReplayArgs {
    FrameView f;
    bsr_outputs out;
    double bg[3];
    double alpha_min, t_stop;
    const uint32_t *lists;
    const uint2 *ranges;
    // backward only
    const float *d_color, *d_depth;
    bool mask_raw;  // apply d_raw = d_color * [raw >= 0] (full pipeline; core seam gets d_raw)
    // the forward raster's per-entry sub-block masks (frame lists only, else nullptr) and
    // the sub-block geometry of its group count G (raster.cuh TileGrid)
    const uint32_t *emask;
    int mask_w, mask_h, mask_cols;
};

// Entry pre-test: the list entries that can reach this pixel are those whose sub-block mask
// (kept by the forward raster, raster.cuh entry_tile_mask: conservative for the fp64
// alpha >= alpha_min decision, which the fp32 raster relies on for every pixel it
// certifies) has the pixel's sub-block bit; entries past the tile's mask_end were not
// reached by the forward and are all kept.  gather_entries collects, in list order, the
// next survivors from `base` on into surv[] (NT of them, or all that are left) and advances
// base past the last one taken; returns the count.  Uniform across the CTA (called by all
// threads).
struct MaskTest {
    int mend, bit;
};

__device__ __forceinline__ MaskTest mask_test(const ReplayArgs &a, int tile, int start, int px, int py) {
    MaskTest m;
    m.mend = a.emask ? (int)a.f.mask_end[tile] : start;
    m.bit = ((py % BSR_TILE) / a.mask_h) * a.mask_cols + (px % BSR_TILE) / a.mask_w;
    return m;
}

template <int NT>
__device__ __forceinline__ int gather_entries(const ReplayArgs &a, const MaskTest mt, int &base, int end, int *surv, int (*gwc)[NT / 32],
                                              int *next) {
    constexpr int NW = NT / 32;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int n = 0, it = 0;
    while (n < NT && base < end) {
        const int e = base + t;
        bool pass = e < end;
        if (pass && e < mt.mend) pass = (__ldg(a.emask + e) >> mt.bit) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        int *wc = gwc[it & 1];  // double-buffered: no second barrier per step
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        int c = lane < NW ? wc[lane] : 0, incl = c;
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int slot = n + __shfl_sync(0xffffffffu, incl - c, warp) + __popc(m & ((1u << lane) - 1u));
        const int total = __shfl_sync(0xffffffffu, incl, NW - 1);
        if (pass && slot < NT) surv[slot] = e;
        if (n + total > NT) {  // full: the next round resumes after the last survivor taken
            if (pass && slot == NT - 1) *next = e + 1;
            __syncthreads();
            base = *next;
            n = NT;
        } else {
            n += total;
            base += NT;
        }
        ++it;
    }
    __syncthreads();
    return n;
}

// This thread's entry of the next round (-1: none), advancing base: when the rest of the
// list fits in one round, the mask test is applied in place (no compaction barriers on
// the short lists of small frames); otherwise the survivors are gathered.  surv aliases
// round-local shared arrays, hence the barrier after reading it.
template <int NT>
__device__ __forceinline__ int next_entry(const ReplayArgs &a, int tile, int start, int px, int py, int &base, int end,
                                          int *surv, int (*gwc)[NT / 32], int *next) {
    const MaskTest mt = mask_test(a, tile, start, px, py);
    if (end - base <= NT) {
        const int e = base + (int)threadIdx.x;
        base = end;
        if (e >= end) return -1;
        return (e >= mt.mend || ((__ldg(a.emask + e) >> mt.bit) & 1u)) ? e : -1;
    }
    const int n = gather_entries<NT>(a, mt, base, end, surv, gwc, next);
    const int e = (int)threadIdx.x < n ? surv[threadIdx.x] : -1;
    __syncthreads();
    return e;
}


// Evaluate alpha exactly as _raster.pyx:107-113 (fp64, no contraction in this TU).
__device__ __forceinline__ double alpha64(const Entry64 &e, int px, int py, double &dx, double &dy,
                                          double &x, double &kernel) {
    dx = px - e.mx;
    dy = py - e.my;
    const double r2 = e.ca * dx * dx + 2.0 * e.cb * dx * dy + e.cc * dy * dy;
    x = fmin(fmax(r2, 0.0), 1.0);
    // outside the support pow(+0, beta > 0) is +0: skip the fp64 pow (same bits)
    kernel = (x == 1.0 && e.beta > 0.0) ? 0.0 : pow(1.0 - x, e.beta);
    return e.o * kernel;
}

// Forward rounds are wider (kReplayFwdThreads entries) and keep only what the recurrence
// reads: alpha (overwritten by the weight alpha * T once T is known) and r, g, b, z.
// Small frames (few flagged pixels, latency-bound) use one 1024-wide CTA per SM; large ones
// (thousands of flagged pixels) 32 one-warp CTAs per SM for more pixels in flight
// (measured, scripts/gpu/ab_env.sh with BSR_REPLAY_NT: config 3 1024 > 256 > 128, config 4 0.54 ms at
// 1024 -> 0.20 at 256 -> 0.15 at 128; after the mask pre-test 0.172 at 128 -> 0.147 at
// 64 -> 0.122 at 32).  BSR_REPLAY_NT overrides for A/B runs.
constexpr int kRecBatch = 8;  // transmittance steps per batch (the stop test runs per batch)
constexpr int64_t kReplayWideMaxPixels = 4 << 20;
template <int NT>
struct ReplayFwdSmem {
    double alpha[NT], val[4][NT];  // val also holds gather_entries' survivors (2 NT ints)
    int entry[NT];
    int warp_cnt[NT / 32];
    int gwc[2][NT / 32], next;
    int n_cand, n_used;
    bool done;
};

// Block-wide ordered compaction of `cand` into slots [0, n): returns this thread's slot.
template <int NT, typename S>
__device__ __forceinline__ int compact_slot(bool cand, S &sm) {
    constexpr int NW = NT / 32;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned m = __ballot_sync(0xffffffffu, cand);
    if (lane == 0) sm.warp_cnt[warp] = __popc(m);
    __syncthreads();
    // exclusive scan of the NW warp counts inside every warp
    int c = lane < NW ? sm.warp_cnt[lane] : 0, incl = c;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int base = __shfl_sync(0xffffffffu, incl - c, warp);
    const int total = __shfl_sync(0xffffffffu, incl, NW - 1);
    if (t == 0) sm.n_cand = total;
    return base + __popc(m & ((1u << lane) - 1u));
}

// The forward replay's per-pixel state for the backward: fp64 (raw, T, last; T and the
// prefix at the split point) by slot; for the raster backward's part (raster_fwd.cu left
// t_final = -T, last = its certified end) the normalised colour behind the split point,
// (raw - prefix) / T, and the clamp bits of the fp64 raw (rasterizer.py:253).
__device__ __forceinline__ void store_split(const ReplayArgs &a, uint32_t slot, int64_t pix, uint32_t last32,
                                            double r0, double r1,
                                            double r2, double dd, double t_acc, int last, double t_flag,
                                            double p0, double p1, double p2, double pd) {
    const FrameView &f = a.f;
    double *st = f.replay_state + 6 * (int64_t)slot;
    st[0] = r0;
    st[1] = r1;
    st[2] = r2;
    st[3] = dd;
    st[4] = t_acc;
    st[5] = (double)last;
    double *sp = f.split_state + 6 * (int64_t)slot;
    sp[0] = t_flag;
    sp[1] = p0;
    sp[2] = p1;
    sp[3] = p2;
    sp[4] = pd;
    const double it = t_flag > 0.0 ? 1.0 / t_flag : 0.0;
    f.bwd_init[pix] = t_flag > 0.0 ? make_float4((float)((r0 - p0) * it), (float)((r1 - p1) * it),
                                                 (float)((r2 - p2) * it), (float)((dd - pd) * it))
                                   : make_float4((float)a.bg[0], (float)a.bg[1], (float)a.bg[2], 0.f);
    f.last[pix] = (last32 & 0x1FFFFFFFu) | (!(r0 >= 0.0) ? 1u << 29 : 0u) | (!(r1 >= 0.0) ? 1u << 30 : 0u) |
                  (!(r2 >= 0.0) ? 1u << 31 : 0u);
}

// One flagged pixel, one CTA: NT list entries per round evaluated in
// parallel (fp64 alpha), then the order-dependent recurrence in two phases: thread 0 runs
// the transmittance chain T <- T * (1 - alpha) over the compacted candidates (batches of
// kRecBatch with no branch inside, the stop test once per batch) and stores each weight
// alpha * T; then lanes 0..3 of warp 0 each carry one of the r, g, b, depth sums over the
// used candidates.  Same operations in the same order as _raster.pyx:95-127.
template <typename P, int NT>
__device__ void replay_fwd_one(const ReplayArgs &a, const P &prov, uint32_t slot, ReplayFwdSmem<NT> &sm) {
    const FrameView &f = a.f;
    const int t = threadIdx.x;
    const uint32_t *lists = a.lists ? a.lists : f.lists;
    const uint2 *ranges = a.ranges ? a.ranges : f.tile_ranges;
    const uint2 fl = f.flags[slot];
    const int64_t pix = fl.x;
    const int px = (int)(pix % f.W), py = (int)(pix / f.W);
    const int tile = (py / BSR_TILE) * f.tiles_x + px / BSR_TILE;
    const int start = (int)ranges[tile].x, end = (int)ranges[tile].y;
    const int flag_at = (int)fl.y;
    const uint32_t last32 = t == 0 ? f.last[pix] : 0u;  // the fp32 part's end (raster_fwd.cu), read early

    double t_acc = 1.0;  // thread 0: transmittance
    double sum = 0.0;    // lane c < 4 of warp 0: running r / g / b / depth sum
    // at the first candidate at/after the fp32 flag point: T (thread 0) and the sums (lanes
    // 0..3) before it -- the backward's split point (raster_bwd takes the entries before it)
    double t_flag = 0.0, pre = 0.0;
    bool flag_open = true;  // uniform: the flag point was not passed yet
    int count = 0, last = 0;
    if (t == 0) sm.done = false;
    __syncthreads();
    int *surv = reinterpret_cast<int *>(&sm.val[0][0]);
    int base = start;
    while (base < end) {
        if (sm.done) break;  // uniform (read after a barrier)
        const int e = next_entry<NT>(a, tile, start, px, py, base, end, surv, sm.gwc, &sm.next);
        Entry64 en;
        bool cand = false;
        double alpha = 0.0;
        if (e >= 0 && prov.get(lists[e], px, py, en)) {
            double dx, dy, x, k;
            alpha = alpha64(en, px, py, dx, dy, x, k);
            cand = !(alpha < a.alpha_min);
            if (cand) prov.color(en);
        }
        const int s = compact_slot<NT>(cand, sm);
        if (cand) {
            sm.alpha[s] = alpha;
            sm.val[0][s] = en.r;
            sm.val[1][s] = en.g;
            sm.val[2][s] = en.b;
            sm.val[3][s] = en.z;
            sm.entry[s] = e - start;
        }
        // candidates of this round before the flag point (also the barrier after the stores)
        int qf = __syncthreads_count(flag_open && cand && e - start < flag_at);
        if (!flag_open) qf = -1;
        if (t < 32) {
            const int n = sm.n_cand;
            if (t == 0) {
                int used = n;
                bool stop = false;
                double tq = 0.0;
                for (int q0 = 0; q0 < n; q0 += kRecBatch) {
                    double al[kRecBatch], tb[kRecBatch + 1];
#pragma unroll
                    for (int j = 0; j < kRecBatch; ++j) al[j] = sm.alpha[q0 + j < n ? q0 + j : 0];
                    tb[0] = t_acc;
#pragma unroll
                    for (int j = 0; j < kRecBatch; ++j) tb[j + 1] = tb[j] * (1.0 - al[j]);
                    if (qf >= q0 && qf < q0 + kRecBatch) {
#pragma unroll
                        for (int j = 0; j < kRecBatch; ++j)
                            if (j == qf - q0) tq = tb[j];
                    }
                    unsigned stops = 0;
#pragma unroll
                    for (int j = 0; j < kRecBatch; ++j) {
                        if (q0 + j < n) {
                            sm.alpha[q0 + j] = al[j] * tb[j];  // weight
                            if (tb[j + 1] < a.t_stop) stops |= 1u << j;
                        }
                    }
                    const int valid = n - q0 < kRecBatch ? n - q0 : kRecBatch;
                    const int take = stops ? __ffs(stops) : valid;  // steps applied from this batch
#pragma unroll
                    for (int j = 1; j <= kRecBatch; ++j)
                        if (j == take) t_acc = tb[j];
                    if (stops) {
                        used = q0 + take;
                        stop = true;
                        break;
                    }
                }
                if (qf >= 0 && qf < used) t_flag = tq;
                count += used;
                if (used > 0) last = sm.entry[used - 1] + 1;
                if (stop) sm.done = true;
                sm.n_used = used;
            }
            __syncwarp();
            if (t < 4) {
                const int used = sm.n_used;
                const double *v = sm.val[t];
                if (qf >= 0 && qf < used) {
                    for (int q = 0; q < qf; ++q) sum = sum + sm.alpha[q] * v[q];
                    pre = sum;
                    for (int q = qf; q < used; ++q) sum = sum + sm.alpha[q] * v[q];
                } else {
#pragma unroll 4
                    for (int q = 0; q < used; ++q) sum = sum + sm.alpha[q] * v[q];
                }
            }
        }
        __syncthreads();
        if (qf >= 0 && qf < sm.n_used) flag_open = false;
        // contributions of entries at/after the fp32 flag point (earlier ones were counted)
        if (cand && s < sm.n_used && sm.entry[s] >= flag_at && a.out.contributions)
            atomicAdd(a.out.contributions + en.src, 1);
        __syncthreads();
    }
    if (t >= 32) return;
    if (flag_open) {  // never reached: the split point is the end
        pre = sum;
        t_flag = t_acc;
    }
    const double c0 = __shfl_sync(0xffffffffu, sum, 0), c1 = __shfl_sync(0xffffffffu, sum, 1);
    const double c2 = __shfl_sync(0xffffffffu, sum, 2), dd = __shfl_sync(0xffffffffu, sum, 3);
    const double p0 = __shfl_sync(0xffffffffu, pre, 0), p1 = __shfl_sync(0xffffffffu, pre, 1);
    const double p2 = __shfl_sync(0xffffffffu, pre, 2), pd = __shfl_sync(0xffffffffu, pre, 3);
    if (t != 0) return;
    const double r0 = c0 + a.bg[0] * t_acc, r1 = c1 + a.bg[1] * t_acc, r2 = c2 + a.bg[2] * t_acc;
    if (a.out.raw) {
        a.out.raw[3 * pix] = (float)r0;
        a.out.raw[3 * pix + 1] = (float)r1;
        a.out.raw[3 * pix + 2] = (float)r2;
    }
    if (a.out.color) {
        a.out.color[3 * pix] = (float)fmax(r0, 0.0);
        a.out.color[3 * pix + 1] = (float)fmax(r1, 0.0);
        a.out.color[3 * pix + 2] = (float)fmax(r2, 0.0);
    }
    if (a.out.alpha) a.out.alpha[pix] = (float)(1.0 - t_acc);
    if (a.out.transmittance) a.out.transmittance[pix] = (float)t_acc;
    if (a.out.depth) a.out.depth[pix] = (float)dd;
    if (a.out.pixel_count) a.out.pixel_count[pix] = count;
    store_split(a, slot, pix, last32, r0, r1, r2, dd, t_acc, last, t_flag, p0, p1, p2, pd);
}

// Gradients of one candidate (_raster.pyx:206-241 + depth) from its T and the colour /
// depth prefix before it, added into grad_acc (or the deterministic accumulator).
__device__ __forceinline__ void pair_grad(const ReplayArgs &a, uint32_t c, const Entry64 &en, double alpha, double my_t,
                                          double p0, double p1, double p2, double pd, double raw0, double raw1,
                                          double raw2, double rawd, double g0, double g1, double g2, double gd,
                                          double dx, double dy, double x, double kernel) {
    const FrameView &f = a.f;
    const double weight = alpha * my_t;
    const double cr0 = weight * en.r, cr1 = weight * en.g, cr2 = weight * en.b, crd = weight * en.z;
    const double behind0 = raw0 - p0 - cr0;
    const double behind1 = raw1 - p1 - cr1;
    const double behind2 = raw2 - p2 - cr2;
    const double behindd = rawd - pd - crd;
    const double g_dot_col = g0 * en.r + g1 * en.g + g2 * en.b;
    const double g_dot_behind = g0 * behind0 + g1 * behind1 + g2 * behind2;
    double d_alpha = g_dot_col * my_t - g_dot_behind / (1.0 - alpha);
    d_alpha = d_alpha + (gd * en.z * my_t - gd * behindd / (1.0 - alpha));
    // partial -> slot of primitive c: float atomics, or the deterministic fixed-point
    // accumulator (frame.cuh DetAcc); the float rounding of the value is the same in
    // both, so both modes sum the same terms
    float *acc = f.grad_acc + (int64_t)c * kGradStride;
    auto add = [&](int slot, double v) {
        if (f.det.mode)
            det_add(f.det, c, slot, (double)(float)v);
        else
            atomicAdd(acc + slot, (float)v);
    };
    add(7, weight * g0);
    add(8, weight * g1);
    add(9, weight * g2);
    add(10, weight * gd);
    add(5, d_alpha * kernel);
    const double d_kernel = d_alpha * en.o;
    if (x < 1.0) {
        add(6, d_kernel * kernel * log(1.0 - x));
        double dkdx = -en.beta * pow(1.0 - x, en.beta - 1.0);
        if (dkdx < -1e7) dkdx = -1e7;
        const double d_x = d_kernel * dkdx;
        double l11, l21, l22;
        if (!record_factor64(f, c, l11, l21, l22)) {  // no factor: xy-frame fp64 partials
            add_geom64(f, c, d_x, dx, dy, en.ca, en.cb, en.cc);
        } else {  // whitened frame of the record's factor (frame.cuh grad_acc)
            const double u = l11 * dx + l21 * dy, w = l22 * dy;
            add(0, d_x * u);
            add(1, d_x * w);
            add(2, d_x * u * u);
            add(3, d_x * u * w);
            add(4, d_x * w * w);
        }
    }
}

// Backward of one flagged pixel by one CTA (small frames: few flagged pixels, so the
// latency of one matters): BSR_BLOCK entries per round from the split point on, evaluated
// in parallel; thread 0 computes every candidate's (T, prefix) in order, then the
// per-candidate gradients are evaluated in parallel.  Same operations as the warp version.
struct ReplayBwdSmem {
    double alpha[BSR_BLOCK], r[BSR_BLOCK], g[BSR_BLOCK], b[BSR_BLOCK], z[BSR_BLOCK];  // r: also survivors
    double t_before[BSR_BLOCK], p0[BSR_BLOCK], p1[BSR_BLOCK], p2[BSR_BLOCK], pd[BSR_BLOCK];
    int warp_cnt[BSR_BLOCK / 32];
    int gwc[2][BSR_BLOCK / 32], next;
    int n_cand;
};

template <typename P>
__device__ void replay_bwd_cta(const ReplayArgs &a, const P &prov, uint32_t slot, ReplayBwdSmem &sm) {
    const FrameView &f = a.f;
    const int t = threadIdx.x;
    const uint32_t *lists = a.lists ? a.lists : f.lists;
    const uint2 *ranges = a.ranges ? a.ranges : f.tile_ranges;
    const uint2 fl = f.flags[slot];
    const int64_t pix = fl.x;
    const int px = (int)(pix % f.W), py = (int)(pix / f.W);
    const int tile = (py / BSR_TILE) * f.tiles_x + px / BSR_TILE;
    const int start = (int)ranges[tile].x;
    const double *st = f.replay_state + 6 * (int64_t)slot;
    const int end = start + (int)st[5];
    const int flag_at = (int)fl.y;
    const double raw0 = st[0], raw1 = st[1], raw2 = st[2], rawd = st[3];
    const double g0 = (!a.mask_raw || raw0 >= 0.0) ? (double)a.d_color[3 * pix] : 0.0;
    const double g1 = (!a.mask_raw || raw1 >= 0.0) ? (double)a.d_color[3 * pix + 1] : 0.0;
    const double g2 = (!a.mask_raw || raw2 >= 0.0) ? (double)a.d_color[3 * pix + 2] : 0.0;
    const double gd = a.d_depth ? (double)a.d_depth[pix] : 0.0;
    const double *sp = f.split_state + 6 * (int64_t)slot;
    double t_acc = sp[0], q0 = sp[1], q1 = sp[2], q2 = sp[3], qd = sp[4];  // thread 0's running state
    int *surv = reinterpret_cast<int *>(sm.r);
    int base = start + flag_at;
    while (base < end) {
        const int e = next_entry<BSR_BLOCK>(a, tile, start, px, py, base, end, surv, sm.gwc, &sm.next);
        Entry64 en;
        bool cand = false;
        double alpha = 0.0, dx = 0, dy = 0, x = 1, kernel = 0;
        uint32_t c = 0;
        if (e >= 0) {
            c = lists[e];
            if (prov.get(c, px, py, en)) {
                alpha = alpha64(en, px, py, dx, dy, x, kernel);
                cand = !(alpha < a.alpha_min);
                if (cand) prov.color(en);
            }
        }
        const int s = compact_slot<BSR_BLOCK>(cand, sm);
        if (cand) {
            sm.alpha[s] = alpha;
            sm.r[s] = en.r;
            sm.g[s] = en.g;
            sm.b[s] = en.b;
            sm.z[s] = en.z;
        }
        __syncthreads();
        if (t == 0) {
            for (int q = 0; q < sm.n_cand; ++q) {
                sm.t_before[q] = t_acc;
                sm.p0[q] = q0;
                sm.p1[q] = q1;
                sm.p2[q] = q2;
                sm.pd[q] = qd;
                const double weight = sm.alpha[q] * t_acc;
                q0 = q0 + weight * sm.r[q];
                q1 = q1 + weight * sm.g[q];
                q2 = q2 + weight * sm.b[q];
                qd = qd + weight * sm.z[q];
                t_acc = t_acc * (1.0 - sm.alpha[q]);
            }
        }
        __syncthreads();
        if (cand)
            pair_grad(a, c, en, alpha, sm.t_before[s], sm.p0[s], sm.p1[s], sm.p2[s], sm.pd[s], raw0, raw1, raw2, rawd,
                      g0, g1, g2, gd, dx, dy, x, kernel);
        __syncthreads();
    }
}

// Backward of one flagged pixel (_raster.pyx:182-241 + depth) by one warp, over the entries
// from the split point on (the raster backward took the certified ones before it, see
// store_split): usually a handful, so one warp per pixel and many pixels in flight.  Entries
// in chunks of 32 (one per lane, after the mask pre-test); each candidate's (T, prefix) runs
// over the chunk's candidates in list order, redundantly in every lane, the values taken
// from the candidate's lane by shuffles -- no shared memory, no block barriers.
__device__ __forceinline__ double shfl64(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

template <typename P>
__device__ void replay_bwd_warp(const ReplayArgs &a, const P &prov, uint32_t slot) {
    const FrameView &f = a.f;
    const int lane = threadIdx.x & 31;
    const uint32_t *lists = a.lists ? a.lists : f.lists;
    const uint2 *ranges = a.ranges ? a.ranges : f.tile_ranges;
    const uint2 fl = f.flags[slot];
    const int64_t pix = fl.x;
    const int px = (int)(pix % f.W), py = (int)(pix / f.W);
    const int tile = (py / BSR_TILE) * f.tiles_x + px / BSR_TILE;
    const int start = (int)ranges[tile].x;
    const double *st = f.replay_state + 6 * (int64_t)slot;
    const int end = start + (int)st[5];
    const int flag_at = (int)fl.y;  // entries before it: raster_bwd (bwd_init)
    if (start + flag_at >= end) return;
    const double raw0 = st[0], raw1 = st[1], raw2 = st[2], rawd = st[3];
    const double g0 = (!a.mask_raw || raw0 >= 0.0) ? (double)a.d_color[3 * pix] : 0.0;
    const double g1 = (!a.mask_raw || raw1 >= 0.0) ? (double)a.d_color[3 * pix + 1] : 0.0;
    const double g2 = (!a.mask_raw || raw2 >= 0.0) ? (double)a.d_color[3 * pix + 2] : 0.0;
    const double gd = a.d_depth ? (double)a.d_depth[pix] : 0.0;
    const MaskTest mt = mask_test(a, tile, start, px, py);
    const double *sp = f.split_state + 6 * (int64_t)slot;
    double t_acc = sp[0], q0 = sp[1], q1 = sp[2], q2 = sp[3], qd = sp[4];
    for (int base = start + flag_at; base < end; base += 32) {
        const int e = base + lane;
        bool pass = e < end;
        if (pass && e < mt.mend) pass = (__ldg(a.emask + e) >> mt.bit) & 1u;
        Entry64 en;
        bool cand = false;
        double alpha = 0.0, dx = 0, dy = 0, x = 1, kernel = 0;
        uint32_t c = 0;
        if (pass) {
            c = lists[e];
            if (prov.get(c, px, py, en)) {
                alpha = alpha64(en, px, py, dx, dy, x, kernel);
                cand = !(alpha < a.alpha_min);
                if (cand) prov.color(en);
            }
        }
        unsigned cm = __ballot_sync(0xffffffffu, cand);
        double my_t = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0, md = 0.0;
        while (cm) {
            const int src = __ffs(cm) - 1;
            cm &= cm - 1u;
            const double al = shfl64(alpha, src);
            const double r = shfl64(en.r, src), g = shfl64(en.g, src), b = shfl64(en.b, src), z = shfl64(en.z, src);
            if (lane == src) {
                my_t = t_acc;
                m0 = q0;
                m1 = q1;
                m2 = q2;
                md = qd;
            }
            const double weight = al * t_acc;
            q0 = q0 + weight * r;
            q1 = q1 + weight * g;
            q2 = q2 + weight * b;
            qd = qd + weight * z;
            t_acc = t_acc * (1.0 - al);
        }
        if (cand)
            pair_grad(a, c, en, alpha, my_t, m0, m1, m2, md, raw0, raw1, raw2, rawd, g0, g1, g2, gd, dx, dy, x, kernel);
    }
}

template <typename P>
__global__ void __launch_bounds__(BSR_BLOCK) replay_bwd_cta_kernel(ReplayArgs a, P prov) {
    pdl_wait();
    __shared__ ReplayBwdSmem sm;
    const uint32_t n = a.f.ctr->flagged;
    for (uint32_t slot = blockIdx.x; slot < n; slot += gridDim.x) {
        replay_bwd_cta(a, prov, slot, sm);
        __syncthreads();
    }
}

template <typename P>
__global__ void __launch_bounds__(BSR_BLOCK, 2) replay_bwd_warp_kernel(ReplayArgs a, P prov) {
    pdl_wait();
    const uint32_t n = a.f.ctr->flagged;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; slot < n; slot += nw)
        replay_bwd_warp(a, prov, slot);
}

template <typename P, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) replay_fwd_kernel(ReplayArgs a, P prov) {
    pdl_wait();
    __shared__ ReplayFwdSmem<NT> sm;
    const uint32_t n = a.f.ctr->flagged;
    for (uint32_t slot = blockIdx.x; slot < n; slot += gridDim.x) {
        replay_fwd_one<P, NT>(a, prov, slot, sm);
        __syncthreads();
    }
}

int raster_groups();

template <typename P>
static int launch_replay(bool fwd, const ReplayArgs &a, const P &prov, cudaStream_t st) {
    if (fwd)
    {
        static const int nt_env = [] {
            const char *e = getenv("BSR_REPLAY_NT");
            return e ? atoi(e) : 0;
        }();
        const int nt = nt_env ? nt_env : ((int64_t)a.f.W * a.f.H <= kReplayWideMaxPixels ? 1024 : 32);
        switch (nt) {
            case 1024: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 1024>, dim3(148), dim3(1024), 0, st, a, prov))); break;
            case 512: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 512>, dim3(2 * 148), dim3(512), 0, st, a, prov))); break;
            case 256: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 256>, dim3(4 * 148), dim3(256), 0, st, a, prov))); break;
            case 128: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 128>, dim3(8 * 148), dim3(128), 0, st, a, prov))); break;
            case 64: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 64>, dim3(16 * 148), dim3(64), 0, st, a, prov))); break;
            default: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 32>, dim3(32 * 148), dim3(32), 0, st, a, prov))); break;
        }
    }
    else if ((int64_t)a.f.W * a.f.H <= kReplayWideMaxPixels)  // one CTA per flagged pixel
        BSR_CUDA_TRY((pdl_launch(replay_bwd_cta_kernel<P>, dim3(2 * 148), dim3(BSR_BLOCK), 0, st, a, prov)));
    else  // one warp per flagged pixel, 8 per CTA, grid-stride over the device-side count
        BSR_CUDA_TRY((pdl_launch(replay_bwd_warp_kernel<P>, dim3(2 * 148), dim3(BSR_BLOCK), 0, st, a, prov)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

int launch_replay_scene(bool fwd, const FrameView &f, const bsr_scene &sc, const KCam &cam,
                        const bsr_outputs &out, const double bg[3], double alpha_min, double t_stop,
                        const float *d_color, const float *d_depth, cudaStream_t st) {
    ReplayArgs a;
    a.f = f;
    a.out = out;
    for (int i = 0; i < 3; ++i) a.bg[i] = bg[i];
    a.alpha_min = alpha_min;
    a.t_stop = t_stop;
    a.lists = nullptr;
    a.ranges = nullptr;
    a.d_color = d_color;
    a.d_depth = d_depth;
    a.mask_raw = true;
    a.emask = f.entry_cap > 0 ? f.emask : nullptr;  // the frame's own lists
    const int g = raster_groups();
    a.mask_w = g == 1 ? 8 : 4;
    a.mask_h = g == 4 ? 2 : 4;
    a.mask_cols = BSR_TILE / a.mask_w;
    int rc = BSR_OK;
#define BSR_REPLAY_LAUNCH(CM) rc = launch_replay(fwd, a, SceneProvider<CM>{sc, cam, f.rec, f.rec64}, st)
    BSR_DISPATCH_CM(sc, BSR_REPLAY_LAUNCH);
#undef BSR_REPLAY_LAUNCH
    return rc;
}

int launch_replay_arrays(bool fwd, const FrameView &f, const double *means, const double *conics,
                         const double *opac, const double *betas, const double *colors,
                         const int32_t *bounds, const uint32_t *lists, const uint2 *ranges,
                         const bsr_outputs &out, const double bg[3], double alpha_min,
                         double t_stop, const float *d_raw, cudaStream_t st) {
    ReplayArgs a;
    a.f = f;
    a.out = out;
    for (int i = 0; i < 3; ++i) a.bg[i] = bg[i];
    a.alpha_min = alpha_min;
    a.t_stop = t_stop;
    a.lists = lists;
    a.ranges = ranges;
    a.d_color = d_raw;
    a.d_depth = nullptr;
    a.mask_raw = false;
    a.emask = nullptr;  // the caller's lists: no forward masks
    a.mask_w = a.mask_h = a.mask_cols = 1;
    ArrayProvider p{means, conics, opac, betas, colors, bounds};
    return launch_replay(fwd, a, p, st);
}

}  // namespace bsr
