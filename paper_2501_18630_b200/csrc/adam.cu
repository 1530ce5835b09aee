// K8: fused Adam over one flat parameter buffer with per-group learning rates
// (training.py:258-273: beta1 .9, beta2 .999, eps 1e-15, bias correction
//  p -= lr * (m / c1) / (sqrt(v / c2) + eps)).
// HBM roofline: 28 B per parameter (p, g, m, v read; p, m, v written).
#include <math.h>

#include "common.cuh"

namespace bsr {

constexpr int kMaxGroups = 16;

struct AdamArgs {
    float *p, *m, *v;
    const float *g;
    int64_t count;
    int n_groups;
    int64_t end[kMaxGroups];
    float lr[kMaxGroups];
    float b1, b2, omb1, omb2, inv_c1, inv_c2, eps;
    const int64_t *step_dev;  // device step counter (graph-capturable variant) or nullptr
    double beta1, beta2;
    int sched_group;  // group whose lr follows `sched` at the device step (-1: none)
    bsr_lr_schedule sched;
    unsigned long long *ticket;  // in-kernel step bump: the last block to finish increments
    float *gzero;                // gradients to clear after use (fused zeroing), or nullptr
};

// training.exponential_lr (training.py:134-145) x scene scale
__device__ inline double adam_sched_lr(const bsr_lr_schedule &s, double step) {
    double t = fmin(fmax(step / (double)s.max_steps, 0.0), 1.0);
    double lr = exp((1.0 - t) * log(s.lr_init) + t * log(s.lr_final));
    if (s.delay_steps > 0) {
        const double u = fmin(fmax(step / (double)s.delay_steps, 0.0), 1.0);
        lr *= s.delay_mult + (1.0 - s.delay_mult) * sin(0.5 * 3.141592653589793 * u);
    }
    return s.scale * lr;
}

__device__ __forceinline__ float group_lr(const AdamArgs &a, int64_t i, float lr_sched) {
    int g = a.n_groups - 1;
    for (int k = a.n_groups - 2; k >= 0; --k)
        if (i < a.end[k]) g = k;
    return g == a.sched_group ? lr_sched : a.lr[g];
}

__device__ __forceinline__ void adam1(const AdamArgs &a, float &p, float g, float &m, float &v,
                                      float lr, float inv_c1, float inv_c2) {
    m = a.b1 * m + a.omb1 * g;
    v = a.b2 * v + a.omb2 * g * g;
    p -= lr * __fdividef(m * inv_c1, sqrtf(v * inv_c2) + a.eps);
}

// Two float4 per thread, all loads issued before any arithmetic (bytes in flight);
// ALIGNED4: every group boundary is a multiple of 4 (the flat 16-byte group layout of
// primitive.py), so one learning rate serves a whole float4.
template <bool ALIGNED4>
__global__ void __launch_bounds__(BSR_BLOCK) adam_kernel(AdamArgs a) {
    pdl_wait();
    __shared__ float s_c[3];
    if (threadIdx.x == 0) {
        float c1 = a.inv_c1, c2 = a.inv_c2, ls = 0.f;
        if (a.step_dev) {  // bias corrections from the device-side step (next value)
            const double st = (double)(*a.step_dev + 1);
            c1 = (float)(1.0 / (1.0 - pow(a.beta1, st)));
            c2 = (float)(1.0 / (1.0 - pow(a.beta2, st)));
            if (a.sched_group >= 0) ls = (float)adam_sched_lr(a.sched, st);
        }
        s_c[0] = c1;
        s_c[1] = c2;
        s_c[2] = ls;
    }
    __syncthreads();
    const float inv_c1 = s_c[0], inv_c2 = s_c[1], lr_s = s_c[2];
    const int64_t n4 = a.count / 4;
    const int64_t q0 = blockIdx.x * (int64_t)(2 * BSR_BLOCK) + threadIdx.x;
    float4 p[2], g[2], m[2], v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int64_t q = q0 + u * BSR_BLOCK;
        if (q < n4) {
            p[u] = reinterpret_cast<const float4 *>(a.p)[q];
            g[u] = reinterpret_cast<const float4 *>(a.g)[q];
            m[u] = reinterpret_cast<const float4 *>(a.m)[q];
            v[u] = reinterpret_cast<const float4 *>(a.v)[q];
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int64_t q = q0 + u * BSR_BLOCK;
        if (q >= n4) continue;
        const int64_t i = 4 * q;
        const float l0 = group_lr(a, i, lr_s);
        adam1(a, p[u].x, g[u].x, m[u].x, v[u].x, l0, inv_c1, inv_c2);
        adam1(a, p[u].y, g[u].y, m[u].y, v[u].y, ALIGNED4 ? l0 : group_lr(a, i + 1, lr_s), inv_c1, inv_c2);
        adam1(a, p[u].z, g[u].z, m[u].z, v[u].z, ALIGNED4 ? l0 : group_lr(a, i + 2, lr_s), inv_c1, inv_c2);
        adam1(a, p[u].w, g[u].w, m[u].w, v[u].w, ALIGNED4 ? l0 : group_lr(a, i + 3, lr_s), inv_c1, inv_c2);
        reinterpret_cast<float4 *>(a.p)[q] = p[u];
        reinterpret_cast<float4 *>(a.m)[q] = m[u];
        reinterpret_cast<float4 *>(a.v)[q] = v[u];
        if (a.gzero) reinterpret_cast<float4 *>(a.gzero)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (blockIdx.x == 0 && threadIdx.x < a.count - 4 * n4) {  // tail (< 4 elements)
        const int64_t i = 4 * n4 + threadIdx.x;
        adam1(a, a.p[i], a.g[i], a.m[i], a.v[i], group_lr(a, i, lr_s), inv_c1, inv_c2);
        if (a.gzero) a.gzero[i] = 0.f;
    }
    if (a.ticket) {  // every block consumed the step above; the last one to get here bumps it
        if (threadIdx.x == 0) {
            if (atomicAdd(a.ticket, 1ull) == gridDim.x - 1) {
                *a.ticket = 0ull;
                *const_cast<int64_t *>(a.step_dev) += 1;
            }
        }
    }
}

__global__ void adam_bump_kernel(int64_t *step) {
    pdl_wait(); *step += 1; }

}  // namespace bsr

using namespace bsr;

static int adam_impl(float *params, const float *grads, float *exp_avg, float *exp_avg_sq, int64_t count,
                     int32_t n_groups, const int64_t *group_end, const float *group_lr, int64_t step,
                     int64_t *step_dev, double beta1, double beta2, double eps, const bsr_lr_schedule *sched,
                     int32_t sched_group, void *stream, bool fused_bump = false, float *gzero = nullptr) {
    if (count < 0 || n_groups < 1 || n_groups > kMaxGroups || (!step_dev && step < 1) || !group_end ||
        !group_lr)
        return BSR_ERR_BAD_ARG;
    if (count == 0) return BSR_OK;
    if (((uintptr_t)params | (uintptr_t)grads | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq) & 15)
        return BSR_ERR_BAD_ARG;
    AdamArgs a;
    a.p = params;
    a.g = grads;
    a.m = exp_avg;
    a.v = exp_avg_sq;
    a.count = count;
    a.n_groups = n_groups;
    for (int k = 0; k < n_groups; ++k) {
        a.end[k] = group_end[k];
        a.lr[k] = group_lr[k];
    }
    a.b1 = (float)beta1;
    a.b2 = (float)beta2;
    a.omb1 = (float)(1.0 - beta1);
    a.omb2 = (float)(1.0 - beta2);
    a.inv_c1 = step_dev ? 1.f : (float)(1.0 / (1.0 - pow(beta1, (double)step)));
    a.inv_c2 = step_dev ? 1.f : (float)(1.0 / (1.0 - pow(beta2, (double)step)));
    a.eps = (float)eps;
    a.step_dev = step_dev;
    a.beta1 = beta1;
    a.beta2 = beta2;
    a.sched_group = -1;
    a.ticket = fused_bump ? reinterpret_cast<unsigned long long *>(step_dev + 1) : nullptr;
    a.gzero = gzero;
    if (sched) {
        if (!step_dev || sched_group < 0 || sched_group >= n_groups || sched->max_steps <= 0 ||
            sched->lr_init <= 0 || sched->lr_final <= 0)
            return BSR_ERR_BAD_ARG;
        a.sched_group = sched_group;
        a.sched = *sched;
    }
    const int64_t n4 = count / 4;
    const unsigned blocks = (unsigned)imax64(1, div_up(imax64(n4, 1), 2 * BSR_BLOCK));
    bool aligned4 = true;
    for (int k = 0; k < n_groups - 1; ++k) aligned4 = aligned4 && (group_end[k] % 4 == 0);
    if (aligned4)
        BSR_CUDA_TRY((pdl_launch(adam_kernel<true>, dim3(blocks), dim3(BSR_BLOCK), 0, (cudaStream_t)stream, a)));
    else
        BSR_CUDA_TRY((pdl_launch(adam_kernel<false>, dim3(blocks), dim3(BSR_BLOCK), 0, (cudaStream_t)stream, a)));
    if (step_dev && !fused_bump)
        BSR_CUDA_TRY((pdl_launch(adam_bump_kernel, dim3(1), dim3(1), 0, (cudaStream_t)stream, step_dev)));
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_adam_step(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                             int64_t count, int32_t n_groups, const int64_t *group_end,
                             const float *group_lr, int64_t step, double beta1, double beta2,
                             double eps, void *stream) {
    return adam_impl(params, grads, exp_avg, exp_avg_sq, count, n_groups, group_end, group_lr, step, nullptr,
                     beta1, beta2, eps, nullptr, -1, stream);
}

extern "C" int bsr_adam_step_device(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                                    int64_t count, int32_t n_groups, const int64_t *group_end,
                                    const float *group_lr, int64_t *step_counter, double beta1,
                                    double beta2, double eps, void *stream) {
    if (!step_counter) return BSR_ERR_BAD_ARG;
    return adam_impl(params, grads, exp_avg, exp_avg_sq, count, n_groups, group_end, group_lr, 0, step_counter,
                     beta1, beta2, eps, nullptr, -1, stream);
}

extern "C" int bsr_adam_step_scheduled(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                                       int64_t count, int32_t n_groups, const int64_t *group_end,
                                       const float *group_lr, int64_t *step_counter,
                                       const bsr_lr_schedule *sched, int32_t sched_group, double beta1,
                                       double beta2, double eps, void *stream) {
    if (!step_counter || !sched) return BSR_ERR_BAD_ARG;
    return adam_impl(params, grads, exp_avg, exp_avg_sq, count, n_groups, group_end, group_lr, 0, step_counter,
                     beta1, beta2, eps, sched, sched_group, stream);
}

extern "C" int bsr_adam_step_fused(float *params, float *grads, float *exp_avg, float *exp_avg_sq, int64_t count,
                                   int32_t n_groups, const int64_t *group_end, const float *group_lr,
                                   int64_t *step_counter, const bsr_lr_schedule *sched, int32_t sched_group,
                                   double beta1, double beta2, double eps, int32_t zero_grads, void *stream) {
    if (!step_counter) return BSR_ERR_BAD_ARG;
    return adam_impl(params, grads, exp_avg, exp_avg_sq, count, n_groups, group_end, group_lr, 0, step_counter, beta1,
                     beta2, eps, sched, sched ? sched_group : -1, stream, true, zero_grads ? grads : nullptr);
}
