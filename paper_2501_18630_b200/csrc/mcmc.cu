// Training-loop neighbours of the hot path, on the device:
//
//   bsr_regularizers      training.loss direct terms            training.py:98-131
//   bsr_inject_noise      training.inject_noise                 training.py:276-292
//                         (+ exponential_lr / position_lr)      training.py:134-145, 206-215
//   bsr_find_dead         mcmc.find_dead                        mcmc.py:32-36
//   bsr_sample_live       the multinomial draw of               mcmc.py:49-70 (plan_relocation),
//                         numpy Generator.choice(live, p=o/sum)  mcmc.py:108-128 (grow)
//   bsr_apply_relocation  mcmc.apply_relocation                 mcmc.py:86-106
//   bsr_grow              mcmc.grow (after the draw)            mcmc.py:108-146
//
// All of them work on the flat, group-major parameter buffer (primitive.group_layout) and
// its Adam moments, are stream ordered and need no host synchronisation; counts that the
// reference returns as Python sizes live in device memory.  The opacity arithmetic of the
// relocation is fp64 like the reference's (compiled with -fmad=false, see Makefile), and
// the draws reproduce numpy's choice() exactly when the caller passes numpy's uniforms
// (cdf = cumsum(p) / cdf[-1]; idx = searchsorted(cdf, u, side="right")).
#include <math.h>

#include "project.cuh"

namespace bsr {

struct Layout {
    int64_t n;
    int n_groups;
    int width[BSR_MAX_GROUPS];
    int64_t start[BSR_MAX_GROUPS];
    int g_pos, g_rot, g_ls, g_op;
    int row;  // floats per primitive over all groups
};

static bool make_layout(const bsr_layout *l, Layout &o) {
    if (!l || l->n < 0 || l->n_groups < 1 || l->n_groups > BSR_MAX_GROUPS) return false;
    o.n = l->n;
    o.n_groups = l->n_groups;
    o.row = 0;
    for (int g = 0; g < l->n_groups; ++g) {
        if (l->width[g] < 0 || l->start[g] < 0) return false;
        o.width[g] = l->width[g];
        o.start[g] = l->start[g];
        o.row += l->width[g];
    }
    o.g_pos = l->g_positions;
    o.g_rot = l->g_rotations;
    o.g_ls = l->g_log_scales;
    o.g_op = l->g_opacity;
    for (int g : {o.g_pos, o.g_rot, o.g_ls, o.g_op})
        if (g < 0 || g >= o.n_groups) return false;
    return o.width[o.g_pos] == 3 && o.width[o.g_rot] == 4 && o.width[o.g_ls] == 3 && o.width[o.g_op] == 1;
}

// ---------------------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so every (seed, counter) draw is
// independent of launch geometry and of graph replay order.
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}
// uniform double in [0, 1) from 53 random bits
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
    return (double)(((uint64_t)(a >> 5) << 26) | (b >> 6)) * (1.0 / 9007199254740992.0);
}

// training.exponential_lr (training.py:134-145) * scene scale, at iteration `step`.
__host__ __device__ inline double scheduled_lr(const bsr_lr_schedule &s, double step) {
    double t = step / (double)s.max_steps;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double lr = exp((1.0 - t) * log(s.lr_init) + t * log(s.lr_final));
    if (s.delay_steps > 0) {
        double u = step / (double)s.delay_steps;
        u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
        lr *= s.delay_mult + (1.0 - s.delay_mult) * sin(0.5 * 3.141592653589793 * u);
    }
    return s.scale * lr;
}

// ---------------------------------------------------------------------------- regularizers
// training.py:112-124: value += lo * sum(o) + ls * sum(s);  d opacity_raw += lo o (1 - o),
// d log_scales += ls * s  (s = exp(log_scale): d/dlog s of s is s).
__global__ void __launch_bounds__(BSR_BLOCK) regularizer_kernel(const float *__restrict__ op,
                                                                 const float *__restrict__ ls, float *g_op,
                                                                 float *g_ls, int64_t n, double lo, double lsc,
                                                                 double *loss) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x; i < 4 * n; i += (int64_t)gridDim.x * BSR_BLOCK) {
        if (i < n) {
            const double o = sigmoid64((double)op[i]);
            if (lo != 0.0) g_op[i] += (float)(lo * o * (1.0 - o));
            acc += lo * o;
        } else {
            const int64_t q = i - n;
            const double s = exp((double)ls[q]);
            if (lsc != 0.0) g_ls[q] += (float)(lsc * s);
            acc += lsc * s;
        }
    }
    if (!loss) return;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double s_acc[BSR_BLOCK / 32];
    if ((threadIdx.x & 31) == 0) s_acc[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < BSR_BLOCK / 32; ++w) t += s_acc[w];
        atomicAdd(loss, t);
    }
}

// ---------------------------------------------------------------------------- noise
struct NoiseArgs {
    float *pos;
    const float *rot, *ls, *op;
    int64_t n;
    double noise_lr, position_lr;
    bsr_lr_schedule sched;
    bool use_sched;
    const int64_t *step;
    const float *eta;
    uint2 key;
    uint32_t offset_lo, offset_hi;
    int32_t *status;
};

// training.py:276-292:  positions += noise_lr * position_lr * (1 - o)^100 * (Sigma eta),
// gate = beta_eval(o, ln 25) = (1 - o)^(4 * 25), Sigma = (R S)(R S)^T (primitive.py:75-80).
__global__ void __launch_bounds__(BSR_BLOCK) noise_kernel(NoiseArgs a) {
    const int64_t i = blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x;
    if (i >= a.n) return;
    const int64_t step = a.step ? *a.step : 0;
    const double lr = a.use_sched ? scheduled_lr(a.sched, (double)step) : a.position_lr;
    const double o = sigmoid64((double)a.op[i]);
    const double om = 1.0 - o;
    const double om2 = om * om, om4 = om2 * om2, om8 = om4 * om4, om16 = om8 * om8;
    const double om32 = om16 * om16, om64 = om32 * om32;
    const double gate = om64 * om32 * om4;  // (1 - o)^100
    double eta[3];
    if (a.eta) {
        eta[0] = a.eta[3 * i];
        eta[1] = a.eta[3 * i + 1];
        eta[2] = a.eta[3 * i + 2];
    } else {  // Box-Muller on two Philox blocks (4 uniforms -> 2 normal pairs)
        const uint4 r = philox4x32(make_uint4((uint32_t)i, (uint32_t)(i >> 32), (uint32_t)step + a.offset_lo,
                                              a.offset_hi), a.key);
        const double u1 = 1.0 - u53(r.x, r.y), u2 = u53(r.z, r.w);
        const double rad = sqrt(-2.0 * log(u1));
        double s2, c2;
        sincospi(2.0 * u2, &s2, &c2);
        const uint4 r2 = philox4x32(make_uint4((uint32_t)i, (uint32_t)(i >> 32) | 0x80000000u,
                                               (uint32_t)step + a.offset_lo, a.offset_hi), a.key);
        const double v1 = 1.0 - u53(r2.x, r2.y), v2 = u53(r2.z, r2.w);
        eta[0] = rad * c2;
        eta[1] = rad * s2;
        eta[2] = sqrt(-2.0 * log(v1)) * cospi(2.0 * v2);
    }
    double R[9];
    if (!quat_to_rot64(a.rot + 4 * i, R)) {
        if (a.status) raise_status(a.status, BSR_ERR_DEGENERATE_QUAT);
        return;
    }
    double s[3];
    for (int k = 0; k < 3; ++k) s[k] = exp((double)a.ls[3 * i + k]);
    // Sigma eta = (R S)((R S)^T eta)
    double w[3];
    for (int k = 0; k < 3; ++k) w[k] = s[k] * (R[k] * eta[0] + R[3 + k] * eta[1] + R[6 + k] * eta[2]);
    const double f = a.noise_lr * lr * gate;
    for (int r = 0; r < 3; ++r) {
        const double d = (R[3 * r] * s[0]) * w[0] + (R[3 * r + 1] * s[1]) * w[1] + (R[3 * r + 2] * s[2]) * w[2];
        a.pos[3 * i + r] = (float)((double)a.pos[3 * i + r] + f * d);
    }
}

// ---------------------------------------------------------------------------- MCMC scratch
// [flags u8 n | pad | block sums f64 | W f64 n]
constexpr int kScanBlock = 2048;  // elements per scan block (256 threads x 8)

struct McmcScratch {
    uint8_t *excluded;
    double *bsum;
    double *W;
    int64_t nb;
};
static uint64_t mcmc_scratch_layout(int64_t n, void *base, McmcScratch *s) {
    const int64_t nb = div_up(imax64(n, 1), kScanBlock);
    uint64_t off = 0;
    const uint64_t o_flags = off;
    off = align_up(off + (uint64_t)imax64(n, 1), 256);
    const uint64_t o_bsum = off;
    off = align_up(off + 8 * (uint64_t)(nb + 1), 256);
    const uint64_t o_w = off;
    off = align_up(off + 8 * (uint64_t)imax64(n, 1), 256);
    if (s) {
        uint8_t *b = (uint8_t *)base;
        s->excluded = b + o_flags;
        s->bsum = (double *)(b + o_bsum);
        s->W = (double *)(b + o_w);
        s->nb = nb;
    }
    return off;
}

// ---------------------------------------------------------------------------- find_dead
// Ordered compaction of {i : sigmoid(opacity_raw[i]) < threshold} (np.nonzero order):
// per-block counts, one-block scan, then ordered writes.
__global__ void __launch_bounds__(BSR_BLOCK) dead_count_kernel(const float *op, int64_t n, double thr,
                                                                double *bsum) {
    int cnt = 0;
    const int64_t b0 = blockIdx.x * (int64_t)kScanBlock;
    for (int k = threadIdx.x; k < kScanBlock; k += BSR_BLOCK) {
        const int64_t i = b0 + k;
        if (i < n) cnt += sigmoid64((double)op[i]) < thr;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    __shared__ int s[BSR_BLOCK / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < BSR_BLOCK / 32; ++w) t += s[w];
        bsum[blockIdx.x] = (double)t;
    }
}

// exclusive scan of nb block values in place (one CTA); total -> bsum[nb] (and *total)
__global__ void __launch_bounds__(1024) block_scan_kernel(double *bsum, int64_t nb, int64_t *total_i64) {
    __shared__ double s_w[32];
    __shared__ double s_carry;
    if (threadIdx.x == 0) s_carry = 0.0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
        const int64_t i = b0 + threadIdx.x;
        const double v = i < nb ? bsum[i] : 0.0;
        double incl = v;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            double w = s_w[lane], wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            s_w[lane] = wi - w;
        }
        __syncthreads();
        const double carry = s_carry;
        if (i < nb) bsum[i] = carry + s_w[warp] + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + s_w[warp] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bsum[nb] = s_carry;
        if (total_i64) *total_i64 = (int64_t)s_carry;
    }
}

__global__ void __launch_bounds__(BSR_BLOCK) dead_write_kernel(const float *op, int64_t n, double thr,
                                                                const double *bsum, int64_t *dead) {
    // each thread owns 8 consecutive elements of the block's 2048
    const int64_t b0 = blockIdx.x * (int64_t)kScanBlock;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t bits = 0;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = b0 + 8 * t + k;
        if (i < n && sigmoid64((double)op[i]) < thr) bits |= 1u << k;
    }
    const int mine = __popc(bits);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ int s_w[BSR_BLOCK / 32];
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    int wexcl = 0;
    for (int w = 0; w < warp; ++w) wexcl += s_w[w];
    int64_t pos = (int64_t)bsum[blockIdx.x] + wexcl + incl - mine;
    for (int k = 0; k < 8; ++k)
        if (bits & (1u << k)) dead[pos++] = b0 + 8 * t + k;
}

// ---------------------------------------------------------------------------- sampling
__global__ void mark_excluded_kernel(uint8_t *flags, const int64_t *idx, const int64_t *count, int64_t cap,
                                     int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x;
    const int64_t c = count ? imin64(*count, cap) : cap;
    if (k < c) {
        const int64_t i = idx[k];
        if (i >= 0 && i < n) flags[i] = 1;
    }
}

__device__ __forceinline__ double live_weight(const float *op, const uint8_t *excl, int64_t i, double thr) {
    const double o = sigmoid64((double)op[i]);
    return (o >= thr && !excl[i]) ? o : 0.0;
}

// per-block sums of the live weights (8 consecutive elements per thread, sequential order)
__global__ void __launch_bounds__(BSR_BLOCK) weight_sum_kernel(const float *op, const uint8_t *excl, int64_t n,
                                                                double thr, double *bsum, int64_t *live_blk) {
    const int64_t b0 = blockIdx.x * (int64_t)kScanBlock;
    double acc = 0.0;
    int live = 0;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = b0 + 8 * threadIdx.x + k;
        if (i < n) {
            const double w = live_weight(op, excl, i, thr);
            acc += w;
            live += w > 0.0;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // ordered (deterministic) block sum: warp inclusive scan, then warp totals in order
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, acc, o);
        if (lane >= o) acc += y;
    }
    live = __reduce_add_sync(0xffffffffu, live);
    __shared__ double s_w[BSR_BLOCK / 32];
    __shared__ int s_l[BSR_BLOCK / 32];
    if (lane == 31) {
        s_w[warp] = acc;
        s_l[warp] = live;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        int l = 0;
        for (int w = 0; w < BSR_BLOCK / 32; ++w) {
            t += s_w[w];
            l += s_l[w];
        }
        bsum[blockIdx.x] = t;
        if (l) atomicAdd((unsigned long long *)live_blk, (unsigned long long)l);
    }
}

// W[i] = inclusive prefix of the live weights / total (the normalised cdf over the full
// index range; non-live entries repeat their predecessor's value)
__global__ void __launch_bounds__(BSR_BLOCK) weight_scan_kernel(const float *op, const uint8_t *excl, int64_t n,
                                                                 double thr, const double *bsum, int64_t nb,
                                                                 double *W) {
    const int64_t b0 = blockIdx.x * (int64_t)kScanBlock;
    double w[8], acc = 0.0;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = b0 + 8 * threadIdx.x + k;
        w[k] = i < n ? live_weight(op, excl, i, thr) : 0.0;
        acc += w[k];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ double s_w[BSR_BLOCK / 32];
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    double run = bsum[blockIdx.x];
    for (int q = 0; q < warp; ++q) run += s_w[q];
    run += incl - acc;
    const double total = bsum[nb];
    const double inv = total > 0.0 ? 1.0 / total : 0.0;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = b0 + 8 * threadIdx.x + k;
        run += w[k];
        if (i < n) W[i] = total > 0.0 ? run * inv : 0.0;
    }
}

// idx = first i with W[i] > u  (== live[searchsorted(cdf, u, side="right")])
__global__ void __launch_bounds__(BSR_BLOCK) draw_kernel(const double *W, int64_t n, const double *uniforms,
                                                          const int64_t *n_draw_dev, int64_t n_draw, uint2 key,
                                                          uint32_t off_lo, uint32_t off_hi, const int64_t *live,
                                                          int64_t *out, int32_t *counts) {
    const int64_t k = blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x;
    const int64_t m = n_draw_dev ? imin64(*n_draw_dev, n_draw) : n_draw;
    if (k >= m || *live == 0) return;
    double u;
    if (uniforms) {
        u = uniforms[k];
    } else {
        const uint4 r = philox4x32(make_uint4((uint32_t)k, (uint32_t)(k >> 32), off_lo, off_hi), key);
        u = u53(r.x, r.y);
    }
    int64_t lo = 0, hi = n;  // first index in [0, n) with W > u
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (W[mid] > u) hi = mid; else lo = mid + 1;
    }
    if (lo >= n) lo = n - 1;  // u >= cdf[-1] cannot happen for u < 1; guard rounding
    out[k] = lo;
    atomicAdd(counts + lo, 1);
}

// ---------------------------------------------------------------------------- relocation
// mcmc.new_opacity + primitive.logit (mcmc.py:73-83, primitive.py:38-41)
__device__ __forceinline__ double adjusted_logit(float op_raw, int mult, double floor_) {
    const double o = sigmoid64((double)op_raw);
    double p = mult == 1 ? o : 1.0 - pow(1.0 - o, 1.0 / (double)mult);
    p = fmax(p, floor_);
    p = fmin(fmax(p, 1e-12), 1.0 - 1e-12);
    return log(p) - log1p(-p);
}

// fp32 storage of an adjusted logit, rounded toward +inf: the reference keeps the fp64
// logit, whose sigmoid clears the floor (e.g. sigmoid(logit(0.005)) >= 0.005), while the
// nearest fp32 can fall just below it and flip the primitive to "dead" in the next draw.
// Rounding up keeps every primitive live that is live in the reference (<= 1 ulp).
__device__ __forceinline__ float stored_logit(double v) { return __double2float_ru(v); }

struct RelocArgs {
    float *p, *m, *v;
    Layout L;
    const int64_t *dead, *targets, *count;
    int64_t cap;
    const int32_t *counts;
    double floor_;
};

// one warp per dead row: copy every group of the target row except the opacity, write the
// adjusted opacity, zero the moments of the dead row
__global__ void __launch_bounds__(BSR_BLOCK) reloc_copy_kernel(RelocArgs a) {
    const int64_t k = (blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t c = imin64(*a.count, a.cap);
    if (k >= c) return;
    const int64_t d = a.dead[k], t = a.targets[k];
    for (int g = 0; g < a.L.n_groups; ++g) {
        const int w = a.L.width[g];
        const int64_t s = a.L.start[g];
        for (int e = lane; e < w; e += 32) {
            float val = a.p[s + w * t + e];
            if (g == a.L.g_op) val = stored_logit(adjusted_logit(val, a.counts[t] + 1, a.floor_));
            a.p[s + w * d + e] = val;
            if (a.m) a.m[s + w * d + e] = 0.f;
            if (a.v) a.v[s + w * d + e] = 0.f;
        }
    }
}

// targets take the same adjusted opacity (read back from any of their copies, which all
// hold the identical value) and zeroed moments
__global__ void __launch_bounds__(BSR_BLOCK) reloc_target_kernel(RelocArgs a) {
    const int64_t k = (blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t c = imin64(*a.count, a.cap);
    if (k >= c) return;
    const int64_t d = a.dead[k], t = a.targets[k];
    const int64_t so = a.L.start[a.L.g_op];
    if (lane == 0) a.p[so + t] = a.p[so + d];
    if (!a.m && !a.v) return;
    for (int g = 0; g < a.L.n_groups; ++g) {
        const int w = a.L.width[g];
        const int64_t s = a.L.start[g];
        for (int e = lane; e < w; e += 32) {
            if (a.m) a.m[s + w * t + e] = 0.f;
            if (a.v) a.v[s + w * t + e] = 0.f;
        }
    }
}

// ---------------------------------------------------------------------------- grow
struct GrowArgs {
    const float *sp, *sm, *sv;
    float *dp, *dm, *dv;
    Layout S, D;
    const int64_t *sources;
    int64_t n_add;
    const int32_t *counts;
    double floor_;
};

// rows [n, n + n_add): copies of their sources with the adjusted opacity; the sources
// themselves (rows [0, n), already copied group-wise by cudaMemcpyAsync) take the same
// opacity and zeroed moments (every copy of a source writes identical values)
__global__ void __launch_bounds__(BSR_BLOCK) grow_rows_kernel(GrowArgs a) {
    const int64_t n = a.S.n;
    const int64_t j = (blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= a.n_add) return;
    const int64_t src = a.sources[j], row = n + j;
    for (int g = 0; g < a.S.n_groups; ++g) {
        const int w = a.S.width[g];
        const int64_t ss = a.S.start[g], ds = a.D.start[g];
        for (int e = lane; e < w; e += 32) {
            float val = a.sp[ss + w * src + e];
            if (g == a.S.g_op) {
                val = stored_logit(adjusted_logit(val, a.counts[src] + 1, a.floor_));
                a.dp[ds + src] = val;
            }
            a.dp[ds + w * row + e] = val;
            if (a.dm) a.dm[ds + w * src + e] = 0.f;
            if (a.dv) a.dv[ds + w * src + e] = 0.f;
        }
    }
}

}  // namespace bsr

using namespace bsr;

static inline uint2 seed_key(uint64_t seed) { return make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)); }

extern "C" int bsr_regularizers(const float *params, const bsr_layout *layout, double lambda_opacity,
                                double lambda_scale, float *grads, double *loss, void *stream) {
    Layout L;
    if (!params || !grads || !make_layout(layout, L)) return BSR_ERR_BAD_ARG;
    if (L.n == 0 || (lambda_opacity == 0.0 && lambda_scale == 0.0)) return BSR_OK;
    const int64_t so = L.start[L.g_op], sl = L.start[L.g_ls];
    const unsigned blocks = (unsigned)imin64(div_up(4 * L.n, BSR_BLOCK), 148 * 8);
    regularizer_kernel<<<blocks, BSR_BLOCK, 0, (cudaStream_t)stream>>>(params + so, params + sl, grads + so,
                                                                        grads + sl, L.n, lambda_opacity,
                                                                        lambda_scale, loss);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_inject_noise(float *params, const bsr_layout *layout, double noise_lr, double position_lr,
                                const bsr_lr_schedule *sched, const int64_t *step_counter, const float *eta,
                                uint64_t seed, uint64_t offset, int32_t *status, void *stream) {
    Layout L;
    if (!params || !make_layout(layout, L)) return BSR_ERR_BAD_ARG;
    if (sched && (!step_counter || sched->max_steps <= 0 || sched->lr_init <= 0 || sched->lr_final <= 0))
        return BSR_ERR_BAD_ARG;
    if (L.n == 0) return BSR_OK;
    NoiseArgs a;
    a.pos = params + L.start[L.g_pos];
    a.rot = params + L.start[L.g_rot];
    a.ls = params + L.start[L.g_ls];
    a.op = params + L.start[L.g_op];
    a.n = L.n;
    a.noise_lr = noise_lr;
    a.position_lr = position_lr;
    a.use_sched = sched != nullptr;
    if (sched) a.sched = *sched;
    a.step = step_counter;
    a.eta = eta;
    a.key = seed_key(seed);
    a.offset_lo = (uint32_t)offset;
    a.offset_hi = (uint32_t)(offset >> 32);
    a.status = status;
    noise_kernel<<<(unsigned)div_up(L.n, BSR_BLOCK), BSR_BLOCK, 0, (cudaStream_t)stream>>>(a);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" double bsr_scheduled_lr(const bsr_lr_schedule *sched, int64_t step) {
    return sched ? scheduled_lr(*sched, (double)step) : 0.0;
}

extern "C" int bsr_mcmc_scratch_bytes(int64_t n, uint64_t *bytes) {
    if (n < 0 || !bytes) return BSR_ERR_BAD_ARG;
    *bytes = mcmc_scratch_layout(n, nullptr, nullptr);
    return BSR_OK;
}

extern "C" int bsr_find_dead(const float *opacity_raw, int64_t n, double threshold, int64_t *dead,
                             int64_t *count, void *scratch, uint64_t scratch_bytes, void *stream) {
    if (n < 0 || !count || (n > 0 && (!opacity_raw || !dead || !scratch))) return BSR_ERR_BAD_ARG;
    if (!(threshold > 0.0 && threshold < 1.0)) return BSR_ERR_BAD_ARG;
    if (scratch_bytes < mcmc_scratch_layout(n, nullptr, nullptr)) return BSR_ERR_FRAME_TOO_SMALL;
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        BSR_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
        return BSR_OK;
    }
    McmcScratch s;
    mcmc_scratch_layout(n, scratch, &s);
    dead_count_kernel<<<(unsigned)s.nb, BSR_BLOCK, 0, st>>>(opacity_raw, n, threshold, s.bsum);
    block_scan_kernel<<<1, 1024, 0, st>>>(s.bsum, s.nb, count);
    dead_write_kernel<<<(unsigned)s.nb, BSR_BLOCK, 0, st>>>(opacity_raw, n, threshold, s.bsum, dead);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_sample_live(const float *opacity_raw, int64_t n, double threshold, const int64_t *exclude,
                               const int64_t *exclude_count, int64_t exclude_cap, const int64_t *n_draw_dev,
                               int64_t n_draw, const double *uniforms, uint64_t seed, uint64_t offset,
                               int64_t *out, int32_t *counts, int64_t *live_count, void *scratch,
                               uint64_t scratch_bytes, void *stream) {
    if (n < 0 || n_draw < 0 || exclude_cap < 0 || !live_count || !counts ||
        (n > 0 && (!opacity_raw || !scratch)) || (n_draw > 0 && !out) || (exclude_cap > 0 && !exclude))
        return BSR_ERR_BAD_ARG;
    if (!(threshold > 0.0 && threshold < 1.0)) return BSR_ERR_BAD_ARG;
    if (scratch_bytes < mcmc_scratch_layout(n, nullptr, nullptr)) return BSR_ERR_FRAME_TOO_SMALL;
    cudaStream_t st = (cudaStream_t)stream;
    BSR_CUDA_TRY(cudaMemsetAsync(live_count, 0, sizeof(int64_t), st));
    if (n == 0) return BSR_OK;
    McmcScratch s;
    mcmc_scratch_layout(n, scratch, &s);
    BSR_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * n, st));
    BSR_CUDA_TRY(cudaMemsetAsync(s.excluded, 0, (size_t)n, st));
    if (exclude_cap > 0)
        mark_excluded_kernel<<<(unsigned)div_up(exclude_cap, BSR_BLOCK), BSR_BLOCK, 0, st>>>(
            s.excluded, exclude, exclude_count, exclude_cap, n);
    weight_sum_kernel<<<(unsigned)s.nb, BSR_BLOCK, 0, st>>>(opacity_raw, s.excluded, n, threshold, s.bsum,
                                                            live_count);
    block_scan_kernel<<<1, 1024, 0, st>>>(s.bsum, s.nb, nullptr);
    weight_scan_kernel<<<(unsigned)s.nb, BSR_BLOCK, 0, st>>>(opacity_raw, s.excluded, n, threshold, s.bsum, s.nb,
                                                             s.W);
    if (n_draw > 0)
        draw_kernel<<<(unsigned)div_up(n_draw, BSR_BLOCK), BSR_BLOCK, 0, st>>>(
            s.W, n, uniforms, n_draw_dev, n_draw, seed_key(seed), (uint32_t)offset, (uint32_t)(offset >> 32),
            live_count, out, counts);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_apply_relocation(float *params, const bsr_layout *layout, float *exp_avg, float *exp_avg_sq,
                                    const int64_t *dead, const int64_t *targets, const int64_t *dead_count,
                                    int64_t dead_cap, const int32_t *counts, double floor_, void *stream) {
    Layout L;
    if (!params || !make_layout(layout, L) || dead_cap < 0 || !dead_count || !counts) return BSR_ERR_BAD_ARG;
    if (dead_cap == 0) return BSR_OK;
    if (!dead || !targets) return BSR_ERR_BAD_ARG;
    RelocArgs a;
    a.p = params;
    a.m = exp_avg;
    a.v = exp_avg_sq;
    a.L = L;
    a.dead = dead;
    a.targets = targets;
    a.count = dead_count;
    a.cap = dead_cap;
    a.counts = counts;
    a.floor_ = floor_;
    const unsigned blocks = (unsigned)div_up(dead_cap * 32, BSR_BLOCK);
    reloc_copy_kernel<<<blocks, BSR_BLOCK, 0, (cudaStream_t)stream>>>(a);
    reloc_target_kernel<<<blocks, BSR_BLOCK, 0, (cudaStream_t)stream>>>(a);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_grow(const float *src_params, const bsr_layout *src_layout, const float *src_exp_avg,
                        const float *src_exp_avg_sq, float *dst_params, const bsr_layout *dst_layout,
                        float *dst_exp_avg, float *dst_exp_avg_sq, const int64_t *sources, int64_t n_add,
                        const int32_t *counts, double floor_, void *stream) {
    Layout S, D;
    if (!src_params || !dst_params || !make_layout(src_layout, S) || !make_layout(dst_layout, D) || !counts ||
        n_add < 0 || (n_add > 0 && !sources))
        return BSR_ERR_BAD_ARG;
    if (D.n != S.n + n_add || D.n_groups != S.n_groups || D.g_op != S.g_op) return BSR_ERR_BAD_ARG;
    for (int g = 0; g < S.n_groups; ++g)
        if (S.width[g] != D.width[g]) return BSR_ERR_BAD_ARG;
    if ((!src_exp_avg) != (!dst_exp_avg) || (!src_exp_avg_sq) != (!dst_exp_avg_sq)) return BSR_ERR_BAD_ARG;
    if (D.n == 0) return BSR_OK;
    GrowArgs a;
    a.sp = src_params;
    a.sm = src_exp_avg;
    a.sv = src_exp_avg_sq;
    a.dp = dst_params;
    a.dm = dst_exp_avg;
    a.dv = dst_exp_avg_sq;
    a.S = S;
    a.D = D;
    a.sources = sources;
    a.n_add = n_add;
    a.counts = counts;
    a.floor_ = floor_;
    cudaStream_t st = (cudaStream_t)stream;
    for (int g = 0; g < S.n_groups; ++g) {
        const size_t old_b = sizeof(float) * (size_t)S.width[g] * (size_t)S.n;
        const size_t add_b = sizeof(float) * (size_t)S.width[g] * (size_t)n_add;
        if (old_b) {
            BSR_CUDA_TRY(cudaMemcpyAsync(dst_params + D.start[g], src_params + S.start[g], old_b,
                                         cudaMemcpyDeviceToDevice, st));
            if (dst_exp_avg)
                BSR_CUDA_TRY(cudaMemcpyAsync(dst_exp_avg + D.start[g], src_exp_avg + S.start[g], old_b,
                                             cudaMemcpyDeviceToDevice, st));
            if (dst_exp_avg_sq)
                BSR_CUDA_TRY(cudaMemcpyAsync(dst_exp_avg_sq + D.start[g], src_exp_avg_sq + S.start[g], old_b,
                                             cudaMemcpyDeviceToDevice, st));
        }
        if (add_b) {
            const int64_t off = D.start[g] + (int64_t)S.width[g] * S.n;
            if (dst_exp_avg) BSR_CUDA_TRY(cudaMemsetAsync(dst_exp_avg + off, 0, add_b, st));
            if (dst_exp_avg_sq) BSR_CUDA_TRY(cudaMemsetAsync(dst_exp_avg_sq + off, 0, add_b, st));
        }
    }
    if (n_add > 0)
        grow_rows_kernel<<<(unsigned)div_up(n_add * 32, BSR_BLOCK), BSR_BLOCK, 0, st>>>(a);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}
