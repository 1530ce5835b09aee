// K7: training loss (1 - l) * L1 + l * (1 - SSIM) and its image gradient
// (training.py:36-131 with lambda_opacity = lambda_scale = 0).
// SSIM: 11-tap Gaussian window (sigma 1.5), zero padding, separable (training.py:36-48),
// C1 = 0.01^2, C2 = 0.03^2, mean over pixels and channels, analytic gradient
// (training.py:65-83).  Two tiled kernels:
//   ssim_maps: blur a, b, a^2, b^2, ab  -> SSIM map terms d_mu, d_qa, d_qab + partial sums
//   ssim_grad: blur the three term maps -> d_image, with the L1 sign term and (optionally)
//              the clamp chain d_raw = d_image * [raw >= 0] (rasterizer.py:253) fused.
// HBM roofline: ~12 fp32 maps of H*W*3.
#include <math.h>

#include "common.cuh"

namespace bsr {

// Tiles of 32 x 32 outputs with a 5-pixel halo (42 x 42 inputs, rows padded to 44 so every
// 4-pixel group is 16-byte aligned).  The Gaussian blur runs on packed FP32 pairs (FFMA2,
// sm_100): the maps kernel blurs (a, b) and (a^2, b^2) as pairs and a*b as a scalar; the
// gradient kernel blurs (d_mu, d_qa) as a pair and d_qab as a scalar.  Both passes produce
// four adjacent outputs per work item from 14 taps (loaded as 16-byte vectors), so the
// taps and the squares are reused four times; the 32 x 32 tile keeps the halo overhead of
// the horizontal pass at 42 / 32 rows.
constexpr int kTW = 32, kTH = 32, kHalo = 5;
constexpr int kIW = kTW + 2 * kHalo, kIH = kTH + 2 * kHalo;  // 42 x 42
constexpr int kIWP = 44;                                      // padded row (16-B aligned quads)
constexpr int kQuads = kTW / 4;                               // 4-output items per row

struct LossArgs {
    const float *a, *b, *raw;
    float2 *pq;               // scratch planes [3][H][W]: (d_mu, d_qa)
    float *px;                // scratch planes [3][H][W]: d_qab
    float *d_image;
    double *sums;             // [2][nblocks]: per-block sums of the ssim map and |a - b|
    int nblocks;
    double *loss_out;         // [3]
    int W, H;
    float w[11];
    double lambda;
};

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

// 4 / 8-byte cp.async with zero fill (src_bytes = 0 -> the destination is zeroed)
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void *smem, const void *gmem, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES),
                 "r"(ok ? BYTES : 0));
}
__device__ __forceinline__ void cp_async_commit_l() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_l() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 14 consecutive float2 (7 x 16 B) / float (4 x 16 B, the last two unused) from shared memory
__device__ __forceinline__ void load14(const float2 *src, float2 (&v)[14]) {
    const float4 *q = reinterpret_cast<const float4 *>(src);
#pragma unroll
    for (int m = 0; m < 7; ++m) {
        const float4 u = q[m];
        v[2 * m] = make_float2(u.x, u.y);
        v[2 * m + 1] = make_float2(u.z, u.w);
    }
}
__device__ __forceinline__ void load14(const float *src, float (&v)[14]) {
    const float4 *q = reinterpret_cast<const float4 *>(src);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const float4 u = q[m];
        if (4 * m < 14) v[4 * m] = u.x;
        if (4 * m + 1 < 14) v[4 * m + 1] = u.y;
        if (4 * m + 2 < 14) v[4 * m + 2] = u.z;
        if (4 * m + 3 < 14) v[4 * m + 3] = u.w;
    }
}

// NC = channels per CTA: 3 (one CTA per tile), or 1 (grid.z = channel: three times the
// CTAs in flight, ~40 KB of shared memory each -- small frames, where one wave of tiles is
// latency-bound; measured: config 1 loss 0.053 -> 0.047 ms, config 4 0.477 -> 0.495 ms)
template <int NC>
struct MapsSmem {
    float2 in[NC][kIH][kIWP];  // (a, b) per channel, zero outside the image
    float2 hp[kIH][kTW], hq[kIH][kTW];
    float hx[kIH][kTW];
    double red[2][8];
};
template <int NC>
struct GradSmem {
    static constexpr int NB = NC == 1 ? 1 : 2;
    float2 p[NB][kIH][kIWP];  // (d_mu, d_qa), double-buffered over channels
    float x[NB][kIH][kIWP];   // d_qab
    float2 hp[kIH][kTW];
    float hx[kIH][kTW];
};

template <int NC>
__global__ void __launch_bounds__(256, NC == 1 ? 4 : 3) ssim_maps_kernel(LossArgs p) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char loss_smem[];
    MapsSmem<NC> &sm = *reinterpret_cast<MapsSmem<NC> *>(loss_smem);
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH, t = threadIdx.x;
    if (NC == 1) {
        // rows of kIW pixels of channel blockIdx.z: six rows per pass
        if (t < 6 * kIW) {
            const int lrow = t / kIW, xx = t - lrow * kIW, gx = x0 - kHalo + xx, c = blockIdx.z;
            const bool okx = gx >= 0 && gx < p.W;
#pragma unroll
            for (int r = lrow; r < kIH; r += 6) {
                const int gy = y0 - kHalo + r;
                const bool ok = okx && gy >= 0 && gy < p.H;
                const int64_t o = ok ? ((int64_t)gy * p.W + gx) * 3 + c : 0;
                cp_async_zfill<4>(&sm.in[0][r][xx].x, p.a + o, ok);
                cp_async_zfill<4>(&sm.in[0][r][xx].y, p.b + o, ok);
            }
        }
    } else if (t < 2 * 3 * kIW) {
        // rows of kIW pixels x 3 channels = 126 contiguous floats: two rows per pass
        // (asynchronous copies: all rows in flight at once, zero fill outside the image)
        const int half = t / (3 * kIW), q = t - half * 3 * kIW;
        const int c = q % 3, xx = q / 3, gx = x0 - kHalo + xx;
        const bool okx = gx >= 0 && gx < p.W;
#pragma unroll 3
        for (int r = half; r < kIH; r += 2) {
            const int gy = y0 - kHalo + r;
            const bool ok = okx && gy >= 0 && gy < p.H;
            const int64_t o = ok ? ((int64_t)gy * p.W + gx) * 3 + c : 0;
            cp_async_zfill<4>(&sm.in[c][r][xx].x, p.a + o, ok);
            cp_async_zfill<4>(&sm.in[c][r][xx].y, p.b + o, ok);
        }
    }
    cp_async_commit_l();
    cp_async_wait_l<0>();
    float w[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) w[k] = p.w[k];
    const int tx = t & 31, r0 = 4 * (t >> 5);
    double s_sum = 0.0, l1_sum = 0.0;
    for (int cc = 0; cc < NC; ++cc) {
        const int c = NC == 1 ? (int)blockIdx.z : cc;
        __syncthreads();
        // horizontal pass: item = (row, 4 adjacent outputs)
        for (int it = t; it < kIH * kQuads; it += 256) {
            const int r = it / kQuads, xb = 4 * (it - r * kQuads);
            float2 v[14], sq[14];
            float xp[14];
            load14(&sm.in[cc][r][xb], v);
#pragma unroll
            for (int k = 0; k < 14; ++k) {
                sq[k] = __fmul2_rn(v[k], v[k]);
                xp[k] = v[k].x * v[k].y;
            }
            float2 P[4], Q[4];
            float X[4];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                P[o] = f2(0.f);
                Q[o] = f2(0.f);
                X[o] = 0.f;
            }
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float2 wk = f2(w[k]);
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                    P[o] = __ffma2_rn(wk, v[k + o], P[o]);
                    Q[o] = __ffma2_rn(wk, sq[k + o], Q[o]);
                    X[o] = fmaf(w[k], xp[k + o], X[o]);
                }
            }
            float4 *hp = reinterpret_cast<float4 *>(&sm.hp[r][xb]);
            float4 *hq = reinterpret_cast<float4 *>(&sm.hq[r][xb]);
            hp[0] = make_float4(P[0].x, P[0].y, P[1].x, P[1].y);
            hp[1] = make_float4(P[2].x, P[2].y, P[3].x, P[3].y);
            hq[0] = make_float4(Q[0].x, Q[0].y, Q[1].x, Q[1].y);
            hq[1] = make_float4(Q[2].x, Q[2].y, Q[3].x, Q[3].y);
            *reinterpret_cast<float4 *>(&sm.hx[r][xb]) = make_float4(X[0], X[1], X[2], X[3]);
        }
        __syncthreads();
        // vertical pass: column tx, output rows r0 .. r0 + 3
        float2 P[4], Q[4];
        float X[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            P[u] = f2(0.f);
            Q[u] = f2(0.f);
            X[u] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 14; ++k) {
            const float2 hp = sm.hp[r0 + k][tx], hq = sm.hq[r0 + k][tx];
            const float hx = sm.hx[r0 + k][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k - u >= 0 && k - u < 11) {
                    const float2 wk = f2(w[k - u]);
                    P[u] = __ffma2_rn(wk, hp, P[u]);
                    Q[u] = __ffma2_rn(wk, hq, Q[u]);
                    X[u] = fmaf(w[k - u], hx, X[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int x = x0 + tx, y = y0 + r0 + u;
            if (x >= p.W || y >= p.H) continue;
            const float mu_a = P[u].x, mu_b = P[u].y, qa = Q[u].x, qb = Q[u].y;
            const float qab = X[u];
            const float C1 = 1e-4f, C2 = 9e-4f;
            const float var_b = qb - mu_b * mu_b;
            const float a1 = 2.f * mu_a * mu_b + C1;
            const float a2 = 2.f * (qab - mu_a * mu_b) + C2;
            const float b1 = mu_a * mu_a + mu_b * mu_b + C1;
            const float b2 = (qa - mu_a * mu_a) + var_b + C2;
            // one division: 1 / b1 = b2 ib, 1 / b2 = b1 ib
            const float ib = 1.f / (b1 * b2);
            const float sv = a1 * a2 * ib;
            const float ib1 = b2 * ib, ib2 = b1 * ib;
            const int64_t o = (int64_t)c * p.H * p.W + (int64_t)y * p.W + x;
            p.pq[o] = make_float2(2.f * mu_b * (a2 - a1) * ib - sv * (2.f * mu_a * (ib1 - ib2)), -sv * ib2);
            p.px[o] = 2.f * a1 * ib;
            s_sum += sv;
            const float2 ctr = sm.in[cc][kHalo + r0 + u][kHalo + tx];
            l1_sum += fabsf(ctr.x - ctr.y);
        }
    }
    // block reduction of the two sums
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
        l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
    }
    if ((t & 31) == 0) {
        sm.red[0][t >> 5] = s_sum;
        sm.red[1][t >> 5] = l1_sum;
    }
    __syncthreads();
    if (t == 0) {  // per-block partials (no same-address atomics across 1e3+ blocks)
        double sv = 0, l = 0;
        for (int i = 0; i < 8; ++i) {
            sv += sm.red[0][i];
            l += sm.red[1][i];
        }
        const int blk = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        p.sums[blk] = sv;
        p.sums[p.nblocks + blk] = l;
    }
}

// loss = (1 - lambda) L1 + lambda (1 - SSIM) from the maps kernel's per-block partials
// (run by block (0, 0) of the gradient kernel, which is stream-ordered after all of them)
__device__ __forceinline__ void loss_finish(const LossArgs &p) {
    __shared__ double red[2][8];
    double sv = 0, l = 0;
    for (int i = threadIdx.x; i < p.nblocks; i += 256) {
        sv += p.sums[i];
        l += p.sums[p.nblocks + i];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        l += __shfl_xor_sync(0xffffffffu, l, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sv;
        red[1][threadIdx.x >> 5] = l;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        sv = l = 0;
        for (int i = 0; i < 8; ++i) {
            sv += red[0][i];
            l += red[1][i];
        }
        const double n = 3.0 * p.W * p.H;
        const double ssim = sv / n, l1 = l / n;
        p.loss_out[0] = (1.0 - p.lambda) * l1 + p.lambda * (1.0 - ssim);
        p.loss_out[1] = l1;
        p.loss_out[2] = ssim;
    }
}

template <int NC>
__global__ void __launch_bounds__(256, NC == 1 ? 4 : 3) ssim_grad_kernel(LossArgs p) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char loss_smem[];
    GradSmem<NC> &sm = *reinterpret_cast<GradSmem<NC> *>(loss_smem);
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH, t = threadIdx.x;
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) loss_finish(p);
    const double n = 3.0 * p.W * p.H;
    const float inv_n = (float)(1.0 / n);
    const float l1w = (float)((1.0 - p.lambda) / n), sw = (float)p.lambda;
    float w[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) w[k] = p.w[k];
    const int tx = t & 31, r0 = 4 * (t >> 5);
    const int lrow = t / kIW, lcol = t - lrow * kIW;  // load mapping: 6 rows of 42 per pass
    const int64_t plane = (int64_t)p.H * p.W;
    auto load_plane = [&](int c, int buf) {
        if (t < 6 * kIW) {
            const int gx = x0 - kHalo + lcol;
            const bool okx = gx >= 0 && gx < p.W;
#pragma unroll
            for (int r = lrow; r < kIH; r += 6) {
                const int gy = y0 - kHalo + r;
                const bool ok = okx && gy >= 0 && gy < p.H;
                const int64_t o = ok ? c * plane + (int64_t)gy * p.W + gx : 0;
                cp_async_zfill<8>(&sm.p[buf][r][lcol], p.pq + o, ok);
                cp_async_zfill<4>(&sm.x[buf][r][lcol], p.px + o, ok);
            }
        }
        cp_async_commit_l();
    };
    load_plane(NC == 1 ? (int)blockIdx.z : 0, 0);
    for (int cc = 0; cc < NC; ++cc) {
        const int c = NC == 1 ? (int)blockIdx.z : cc;
        const int buf = NC == 1 ? 0 : (cc & 1);
        // centre values for the epilogue, in flight during the blur
        float av[4], bv[4], rv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int x = x0 + tx, y = y0 + r0 + q;
            av[q] = bv[q] = 0.f;
            rv[q] = 1.f;
            if (x < p.W && y < p.H) {
                const int64_t o = ((int64_t)y * p.W + x) * 3 + c;
                av[q] = p.a[o];
                bv[q] = p.b[o];
                if (p.raw) rv[q] = p.raw[o];
            }
        }
        __syncthreads();  // buffer buf ^ 1 and hp / hx are free
        if (NC == 3 && cc < 2) {
            load_plane(c + 1, buf ^ 1);
            cp_async_wait_l<1>();
        } else {
            cp_async_wait_l<0>();
        }
        __syncthreads();
        for (int it = t; it < kIH * kQuads; it += 256) {
            const int r = it / kQuads, xb = 4 * (it - r * kQuads);
            float2 v[14];
            float u[14];
            load14(&sm.p[buf][r][xb], v);
            load14(&sm.x[buf][r][xb], u);
            float2 P[4];
            float X[4];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                P[o] = f2(0.f);
                X[o] = 0.f;
            }
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float2 wk = f2(w[k]);
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                    P[o] = __ffma2_rn(wk, v[k + o], P[o]);
                    X[o] = fmaf(w[k], u[k + o], X[o]);
                }
            }
            float4 *hp = reinterpret_cast<float4 *>(&sm.hp[r][xb]);
            hp[0] = make_float4(P[0].x, P[0].y, P[1].x, P[1].y);
            hp[1] = make_float4(P[2].x, P[2].y, P[3].x, P[3].y);
            *reinterpret_cast<float4 *>(&sm.hx[r][xb]) = make_float4(X[0], X[1], X[2], X[3]);
        }
        __syncthreads();
        float2 P[4];
        float X[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            P[q] = f2(0.f);
            X[q] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 14; ++k) {
            const float2 hp = sm.hp[r0 + k][tx];
            const float hx = sm.hx[r0 + k][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (k - q >= 0 && k - q < 11) {
                    P[q] = __ffma2_rn(f2(w[k - q]), hp, P[q]);
                    X[q] = fmaf(w[k - q], hx, X[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int x = x0 + tx, y = y0 + r0 + q;
            if (x >= p.W || y >= p.H) continue;
            const float grad = (P[q].x + 2.f * av[q] * P[q].y + bv[q] * X[q]) * inv_n;
            const float diff = av[q] - bv[q];
            const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
            float d = l1w * sgn - sw * grad;
            if (!(rv[q] >= 0.f)) d = 0.f;
            p.d_image[((int64_t)y * p.W + x) * 3 + c] = d;
        }
    }
}

}  // namespace bsr

using namespace bsr;

extern "C" int bsr_loss_scratch_bytes(int32_t width, int32_t height, uint64_t *bytes) {
    if (!bytes || width < 11 || height < 11) return BSR_ERR_BAD_ARG;
    const uint64_t nb = 3ull * div_up(width, kTW) * div_up(height, kTH);  // at most (NC = 1)
    const uint64_t plane = 3ull * width * height;
    *bytes = align_up(16ull * nb, 256) + align_up(8ull * plane, 256) + align_up(4ull * plane, 256);
    return BSR_OK;
}

template <int NC>
static int launch_loss(const LossArgs &p, cudaStream_t st);
constexpr int64_t kLossSplitMaxPixels = 4 << 20;  // frames up to this size: one channel per CTA

extern "C" int bsr_loss_l1_dssim(const float *rendered, const float *target, const float *raw,
                                 int32_t width, int32_t height, double lambda_ssim, double *loss_out,
                                 float *d_image, void *scratch, uint64_t scratch_bytes, void *stream) {
    uint64_t need = 0;
    if (bsr_loss_scratch_bytes(width, height, &need) != BSR_OK || scratch_bytes < need || !rendered ||
        !target || !d_image || !loss_out || !scratch)
        return BSR_ERR_BAD_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    LossArgs p;
    const uint64_t plane = 3ull * width * height;
    char *base = (char *)scratch;
    const int nc = (int64_t)width * height <= kLossSplitMaxPixels ? 1 : 3;
    p.nblocks = (int)((nc == 1 ? 3 : 1) * div_up(width, kTW) * div_up(height, kTH));
    p.sums = (double *)base;
    p.pq = (float2 *)(base + align_up(16ull * p.nblocks, 256));
    p.px = (float *)((char *)p.pq + align_up(8ull * plane, 256));
    p.a = rendered;
    p.b = target;
    p.raw = raw;
    p.d_image = d_image;
    p.loss_out = loss_out;
    p.W = width;
    p.H = height;
    p.lambda = lambda_ssim;
    double w[11], sum = 0;
    for (int i = 0; i < 11; ++i) {
        const double x = i - 5.0;
        w[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
        sum += w[i];
    }
    for (int i = 0; i < 11; ++i) p.w[i] = (float)(w[i] / sum);
    return nc == 1 ? launch_loss<1>(p, st) : launch_loss<3>(p, st);
}

template <int NC>
static int launch_loss(const LossArgs &p, cudaStream_t st) {
    dim3 grid((unsigned)div_up(p.W, kTW), (unsigned)div_up(p.H, kTH), NC == 1 ? 3u : 1u);
    static SmemAttrOnce attr_maps, attr_grad;
    BSR_CUDA_TRY(attr_maps.ensure(ssim_maps_kernel<NC>, sizeof(MapsSmem<NC>)));
    BSR_CUDA_TRY(attr_grad.ensure(ssim_grad_kernel<NC>, sizeof(GradSmem<NC>)));
    BSR_CUDA_TRY((pdl_launch(ssim_maps_kernel<NC>, dim3(grid), dim3(256), sizeof(MapsSmem<NC>), st, p)));
    BSR_CUDA_TRY((pdl_launch(ssim_grad_kernel<NC>, dim3(grid), dim3(256), sizeof(GradSmem<NC>), st, p)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}
