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

constexpr int kLT = 16;           // output tile edge
constexpr int kHalo = 5;
constexpr int kLI = kLT + 2 * kHalo;  // 26

struct LossArgs {
    const float *a, *b, *raw;
    float *dmu, *dqa, *dqab;  // scratch maps (H,W,3)
    float *d_image;
    double *sums;             // [2][nblocks]: per-block sums of the ssim map and |a - b|
    int nblocks;
    double *loss_out;         // [3]
    int W, H;
    float w[11];
    double lambda;
};

__global__ void __launch_bounds__(256, 4) ssim_maps_kernel(LossArgs p) {
    __shared__ float sa[3][kLI][kLI], sb[3][kLI][kLI];
    __shared__ float h[5][kLI][kLT];
    __shared__ double red[2][8];
    const int tx0 = blockIdx.x * kLT, ty0 = blockIdx.y * kLT;
    const int t = threadIdx.x, lx = t % kLT, ly = t / kLT;
    const int x = tx0 + lx, y = ty0 + ly;
    const bool in = x < p.W && y < p.H;
    double s_sum = 0.0, l1_sum = 0.0;
    // all three channels of the halo tile at once: one global-latency exposure per block
    for (int i = t; i < kLI * kLI * 3; i += 256) {
        const int px = i / 3, c = i - px * 3;
        const int yy = ty0 - kHalo + px / kLI, xx = tx0 - kHalo + px % kLI;
        const bool ok = xx >= 0 && yy >= 0 && xx < p.W && yy < p.H;
        const int64_t o = ((int64_t)yy * p.W + xx) * 3 + c;
        sa[c][px / kLI][px % kLI] = ok ? p.a[o] : 0.f;
        sb[c][px / kLI][px % kLI] = ok ? p.b[o] : 0.f;
    }
    for (int c = 0; c < 3; ++c) {
        __syncthreads();
        // horizontal pass over all kLI rows, kLT output columns
        for (int i = t; i < kLI * kLT; i += 256) {
            const int r = i / kLT, col = i % kLT;
            float m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float av = sa[c][r][col + k], bv = sb[c][r][col + k], wk = p.w[k];
                m0 += wk * av;
                m1 += wk * bv;
                m2 += wk * av * av;
                m3 += wk * bv * bv;
                m4 += wk * av * bv;
            }
            h[0][r][col] = m0;
            h[1][r][col] = m1;
            h[2][r][col] = m2;
            h[3][r][col] = m3;
            h[4][r][col] = m4;
        }
        __syncthreads();
        float mu_a = 0, mu_b = 0, qa = 0, qb = 0, qab = 0;
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const float wk = p.w[k];
            mu_a += wk * h[0][ly + k][lx];
            mu_b += wk * h[1][ly + k][lx];
            qa += wk * h[2][ly + k][lx];
            qb += wk * h[3][ly + k][lx];
            qab += wk * h[4][ly + k][lx];
        }
        if (in) {
            const float C1 = 1e-4f, C2 = 9e-4f;
            const float var_b = qb - mu_b * mu_b;
            const float a1 = 2.f * mu_a * mu_b + C1;
            const float a2 = 2.f * (qab - mu_a * mu_b) + C2;
            const float b1 = mu_a * mu_a + mu_b * mu_b + C1;
            const float b2 = (qa - mu_a * mu_a) + var_b + C2;
            const float ib = 1.f / (b1 * b2);
            const float s = a1 * a2 * ib;
            const int64_t o = ((int64_t)y * p.W + x) * 3 + c;
            p.dmu[o] = 2.f * mu_b * (a2 - a1) * ib - s * (2.f * mu_a / b1 - 2.f * mu_a / b2);
            p.dqa[o] = -s / b2;
            p.dqab[o] = 2.f * a1 * ib;
            s_sum += s;
            l1_sum += fabsf(sa[c][ly + kHalo][lx + kHalo] - sb[c][ly + kHalo][lx + kHalo]);
        }
    }
    // block reduction of the two sums
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
        l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
    }
    if ((t & 31) == 0) {
        red[0][t >> 5] = s_sum;
        red[1][t >> 5] = l1_sum;
    }
    __syncthreads();
    if (t == 0) {  // per-block partials (no same-address atomics across 1e3+ blocks)
        double s = 0, l = 0;
        for (int i = 0; i < 8; ++i) {
            s += red[0][i];
            l += red[1][i];
        }
        const int blk = blockIdx.y * gridDim.x + blockIdx.x;
        p.sums[blk] = s;
        p.sums[p.nblocks + blk] = l;
    }
}

__global__ void __launch_bounds__(256, 4) ssim_grad_kernel(LossArgs p) {
    __shared__ float s[3][3][kLI][kLI];
    __shared__ float h[3][kLI][kLT];
    const int tx0 = blockIdx.x * kLT, ty0 = blockIdx.y * kLT;
    const int t = threadIdx.x, lx = t % kLT, ly = t / kLT;
    const int x = tx0 + lx, y = ty0 + ly;
    const bool in = x < p.W && y < p.H;
    const double n = 3.0 * p.W * p.H;
    const float inv_n = (float)(1.0 / n);
    const float l1w = (float)((1.0 - p.lambda) / n), sw = (float)p.lambda;
    for (int i = t; i < kLI * kLI * 3; i += 256) {
        const int px = i / 3, c = i - px * 3;
        const int yy = ty0 - kHalo + px / kLI, xx = tx0 - kHalo + px % kLI;
        const bool ok = xx >= 0 && yy >= 0 && xx < p.W && yy < p.H;
        const int64_t o = ((int64_t)yy * p.W + xx) * 3 + c;
        s[c][0][px / kLI][px % kLI] = ok ? p.dmu[o] : 0.f;
        s[c][1][px / kLI][px % kLI] = ok ? p.dqa[o] : 0.f;
        s[c][2][px / kLI][px % kLI] = ok ? p.dqab[o] : 0.f;
    }
    for (int c = 0; c < 3; ++c) {
        __syncthreads();
        for (int i = t; i < kLI * kLT; i += 256) {
            const int r = i / kLT, col = i % kLT;
            float m0 = 0, m1 = 0, m2 = 0;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float wk = p.w[k];
                m0 += wk * s[c][0][r][col + k];
                m1 += wk * s[c][1][r][col + k];
                m2 += wk * s[c][2][r][col + k];
            }
            h[0][r][col] = m0;
            h[1][r][col] = m1;
            h[2][r][col] = m2;
        }
        __syncthreads();
        float b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const float wk = p.w[k];
            b0 += wk * h[0][ly + k][lx];
            b1 += wk * h[1][ly + k][lx];
            b2 += wk * h[2][ly + k][lx];
        }
        if (in) {
            const int64_t o = ((int64_t)y * p.W + x) * 3 + c;
            const float av = p.a[o], bv = p.b[o];
            const float grad = (b0 + 2.f * av * b1 + bv * b2) * inv_n;
            const float diff = av - bv;
            const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
            float d = l1w * sgn - sw * grad;
            if (p.raw && !(p.raw[o] >= 0.f)) d = 0.f;
            p.d_image[o] = d;
        }
    }
}

__global__ void __launch_bounds__(256) loss_finish_kernel(LossArgs p) {
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

}  // namespace bsr

using namespace bsr;

extern "C" int bsr_loss_scratch_bytes(int32_t width, int32_t height, uint64_t *bytes) {
    if (!bytes || width < 11 || height < 11) return BSR_ERR_BAD_ARG;
    const uint64_t nb = (uint64_t)div_up(width, kLT) * div_up(height, kLT);
    *bytes = align_up(3ull * 4 * 3 * (uint64_t)width * height, 256) + align_up(16ull * nb, 256);
    return BSR_OK;
}

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
    p.nblocks = (int)(div_up(width, kLT) * div_up(height, kLT));
    p.sums = (double *)base;
    p.dmu = (float *)(base + align_up(16ull * p.nblocks, 256));
    p.dqa = p.dmu + plane;
    p.dqab = p.dqa + plane;
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
    dim3 grid((unsigned)div_up(width, kLT), (unsigned)div_up(height, kLT));
    ssim_maps_kernel<<<grid, 256, 0, st>>>(p);
    ssim_grad_kernel<<<grid, 256, 0, st>>>(p);
    loss_finish_kernel<<<1, 256, 0, st>>>(p);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}
