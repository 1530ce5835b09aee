// fp64 replay of the pixels the fp32 raster could not certify.
//
// For each flagged pixel one warp re-walks the pixel's tile list with the reference's
// fp64 arithmetic (_raster.pyx:101-127 forward, :191-241 backward; this file is compiled
// with -fmad=false like pkg/setup.py's -ffp-contract=off).  Primitive values come from a
// Provider: the full pipeline recomputes them with the same fp64 code as preprocess.cu
// (project.cuh), the core seam reads the caller's fp64 arrays.  Lanes evaluate 32 list
// entries in parallel; the compositing recurrence (order-dependent) runs redundantly in
// every lane over the candidates, in list order.
//
// Forward writes every per-pixel output of the flagged pixel and counts contributions of
// entries at or after the entry where fp32 stopped (entries before it were certified and
// counted by the fp32 kernel).  Backward adds the pixel's gradients into grad_acc.
#include <stdlib.h>

#include "frame.cuh"
#include "appearance.cuh"
#include "project.cuh"
#include "raster.cuh"
#ifdef BSR_REPLAY_TRACE
#include <cstdio>
#endif

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
};

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
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

// Candidates of one round (entries passing alpha >= alpha_min), compacted in list order.
struct ReplaySmem {
    double alpha[BSR_BLOCK], r[BSR_BLOCK], g[BSR_BLOCK], b[BSR_BLOCK], z[BSR_BLOCK];
    double t_before[BSR_BLOCK], p0[BSR_BLOCK], p1[BSR_BLOCK], p2[BSR_BLOCK], pd[BSR_BLOCK];
    int entry[BSR_BLOCK];
    int warp_cnt[BSR_BLOCK / 32];
    int n_cand, n_used;
    bool done;
};

// Forward rounds are wider (kReplayFwdThreads entries) and keep only what the recurrence
// reads: alpha (overwritten by the weight alpha * T once T is known) and r, g, b, z.
// Small frames (few flagged pixels, latency-bound) use one 1024-wide CTA per SM; large ones
// (thousands of flagged pixels) eight 128-wide CTAs per SM for more pixels in flight
// (measured, scripts/ab_replay_nt.sh: config 3 1024 > 256 > 128, config 4 0.54 ms at
// 1024 -> 0.20 at 256 -> 0.15 at 128).  BSR_REPLAY_NT overrides for A/B runs.
constexpr int kRecBatch = 8;  // transmittance steps per batch (the stop test runs per batch)
constexpr int64_t kReplayWideMaxPixels = 4 << 20;
template <int NT>
struct ReplayFwdSmem {
    double alpha[NT], val[4][NT];
    int entry[NT];
    int warp_cnt[NT / 32];
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

    double t_acc = 1.0;  // thread 0: transmittance
    double sum = 0.0;    // lane c < 4 of warp 0: running r / g / b / depth sum
    int count = 0, last = 0;
    if (t == 0) sm.done = false;
    __syncthreads();
#ifdef BSR_REPLAY_TRACE
    long long tr0 = clock64(), tr1 = 0, tr2 = 0;
#endif
    for (int base = start; base < end; base += NT) {
        if (sm.done) break;  // uniform (read after a barrier)
        const int e = base + t;
        Entry64 en;
        bool cand = false;
        double alpha = 0.0;
#ifdef BSR_REPLAY_TRACE
        if (t == 0) tr0 = clock64();
#endif
        if (e < end && prov.get(lists[e], px, py, en)) {
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
        __syncthreads();
#ifdef BSR_REPLAY_TRACE
        if (t == 0) tr1 = clock64();
#endif
        if (t < 32) {
            const int n = sm.n_cand;
            if (t == 0) {
                int used = n;
                bool stop = false;
                for (int q0 = 0; q0 < n; q0 += kRecBatch) {
                    double al[kRecBatch], tb[kRecBatch + 1];
#pragma unroll
                    for (int j = 0; j < kRecBatch; ++j) al[j] = sm.alpha[q0 + j < n ? q0 + j : 0];
                    tb[0] = t_acc;
#pragma unroll
                    for (int j = 0; j < kRecBatch; ++j) tb[j + 1] = tb[j] * (1.0 - al[j]);
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
                count += used;
                if (used > 0) last = sm.entry[used - 1] + 1;
                if (stop) sm.done = true;
                sm.n_used = used;
            }
            __syncwarp();
            if (t < 4) {
                const int used = sm.n_used;
                const double *v = sm.val[t];
#pragma unroll 4
                for (int q = 0; q < used; ++q) sum = sum + sm.alpha[q] * v[q];
            }
        }
        __syncthreads();
#ifdef BSR_REPLAY_TRACE
        if (t == 0) {
            tr2 = clock64();
            printf("replay pix %lld base %d/%d cand %d used %d eval %lld rec %lld\n", (long long)pix, base - start,
                   end - start, sm.n_cand, sm.n_used, tr1 - tr0, tr2 - tr1);
        }
#endif
        // contributions of entries at/after the fp32 flag point (earlier ones were counted)
        if (cand && s < sm.n_used && sm.entry[s] >= flag_at && a.out.contributions)
            atomicAdd(a.out.contributions + en.src, 1);
        __syncthreads();
    }
    if (t >= 32) return;
    const double c0 = __shfl_sync(0xffffffffu, sum, 0), c1 = __shfl_sync(0xffffffffu, sum, 1);
    const double c2 = __shfl_sync(0xffffffffu, sum, 2), dd = __shfl_sync(0xffffffffu, sum, 3);
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
    f.t_final[pix] = (float)t_acc;
    double *st = f.replay_state + 6 * (int64_t)slot;
    st[0] = r0;
    st[1] = r1;
    st[2] = r2;
    st[3] = dd;
    st[4] = t_acc;
    st[5] = (double)last;
}

// Backward of one flagged pixel (_raster.pyx:182-241 + depth), one CTA: parallel alpha,
// thread 0 computes every candidate's (T, prefix) in order, then the per-candidate
// gradients are evaluated in parallel and added into grad_acc.
template <typename P>
__device__ void replay_bwd_one(const ReplayArgs &a, const P &prov, uint32_t slot, ReplaySmem &sm) {
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
    const double raw0 = st[0], raw1 = st[1], raw2 = st[2], rawd = st[3];
    const int end = start + (int)st[5];
    // clamp chain d_raw = d_color * [raw >= 0] on the fp64 raw (rasterizer.py:253)
    const double g0 = (!a.mask_raw || raw0 >= 0.0) ? (double)a.d_color[3 * pix] : 0.0;
    const double g1 = (!a.mask_raw || raw1 >= 0.0) ? (double)a.d_color[3 * pix + 1] : 0.0;
    const double g2 = (!a.mask_raw || raw2 >= 0.0) ? (double)a.d_color[3 * pix + 2] : 0.0;
    const double gd = a.d_depth ? (double)a.d_depth[pix] : 0.0;

    double t_acc = 1.0, q0 = 0.0, q1 = 0.0, q2 = 0.0, qd = 0.0;  // thread 0's running state
    for (int base = start; base < end; base += BSR_BLOCK) {
        const int e = base + t;
        Entry64 en;
        bool cand = false;
        double alpha = 0.0, dx = 0, dy = 0, x = 1, kernel = 0;
        uint32_t c = 0;
        if (e < end) {
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
        if (cand) {
            const double my_t = sm.t_before[s];
            const double weight = alpha * my_t;
            const double cr0 = weight * en.r, cr1 = weight * en.g, cr2 = weight * en.b, crd = weight * en.z;
            const double behind0 = raw0 - sm.p0[s] - cr0;
            const double behind1 = raw1 - sm.p1[s] - cr1;
            const double behind2 = raw2 - sm.p2[s] - cr2;
            const double behindd = rawd - sm.pd[s] - crd;
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
        __syncthreads();
    }
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

template <typename P>
__global__ void __launch_bounds__(BSR_BLOCK) replay_bwd_kernel(ReplayArgs a, P prov) {
    pdl_wait();
    __shared__ ReplaySmem sm;
    const uint32_t n = a.f.ctr->flagged;
    for (uint32_t slot = blockIdx.x; slot < n; slot += gridDim.x) {
        replay_bwd_one(a, prov, slot, sm);
        __syncthreads();
    }
}

static unsigned replay_blocks(const FrameView &) {
    // one CTA per flagged pixel, grid-stride over the device-side count
    return 148 * 2;
}

template <typename P>
static int launch_replay(bool fwd, const ReplayArgs &a, const P &prov, cudaStream_t st) {
    if (fwd)
    {
        static const int nt_env = [] {
            const char *e = getenv("BSR_REPLAY_NT");
            return e ? atoi(e) : 0;
        }();
        const int nt = nt_env ? nt_env : ((int64_t)a.f.W * a.f.H <= kReplayWideMaxPixels ? 1024 : 128);
        switch (nt) {
            case 1024: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 1024>, dim3(148), dim3(1024), 0, st, a, prov))); break;
            case 512: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 512>, dim3(2 * 148), dim3(512), 0, st, a, prov))); break;
            case 256: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 256>, dim3(4 * 148), dim3(256), 0, st, a, prov))); break;
            case 128: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 128>, dim3(8 * 148), dim3(128), 0, st, a, prov))); break;
            default: BSR_CUDA_TRY((pdl_launch(replay_fwd_kernel<P, 64>, dim3(16 * 148), dim3(64), 0, st, a, prov))); break;
        }
    }
    else
        BSR_CUDA_TRY((pdl_launch(replay_bwd_kernel<P>, dim3(replay_blocks(a.f)), dim3(BSR_BLOCK), 0, st, a, prov)));
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
    ArrayProvider p{means, conics, opac, betas, colors, bounds};
    return launch_replay(fwd, a, p, st);
}

}  // namespace bsr
