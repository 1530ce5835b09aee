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
};

__device__ __forceinline__ float group_lr(const AdamArgs &a, int64_t i) {
    float lr = a.lr[a.n_groups - 1];
    for (int k = a.n_groups - 2; k >= 0; --k)
        if (i < a.end[k]) lr = a.lr[k];
    return lr;
}

__device__ __forceinline__ void adam1(const AdamArgs &a, float &p, float g, float &m, float &v,
                                      float lr) {
    m = a.b1 * m + a.omb1 * g;
    v = a.b2 * v + a.omb2 * g * g;
    p -= lr * (m * a.inv_c1) / (sqrtf(v * a.inv_c2) + a.eps);
}

__global__ void __launch_bounds__(BSR_BLOCK) adam_kernel(AdamArgs a) {
    if (a.step_dev) {  // bias corrections from the device-side step (next value)
        const double st = (double)(*a.step_dev + 1);
        a.inv_c1 = (float)(1.0 / (1.0 - pow(a.beta1, st)));
        a.inv_c2 = (float)(1.0 / (1.0 - pow(a.beta2, st)));
    }
    const int64_t n4 = a.count / 4;
    const int64_t stride = (int64_t)gridDim.x * BSR_BLOCK;
    for (int64_t q = blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x; q < n4; q += stride) {
        float4 p = reinterpret_cast<float4 *>(a.p)[q];
        const float4 g = reinterpret_cast<const float4 *>(a.g)[q];
        float4 m = reinterpret_cast<float4 *>(a.m)[q];
        float4 v = reinterpret_cast<float4 *>(a.v)[q];
        const int64_t i = 4 * q;
        adam1(a, p.x, g.x, m.x, v.x, group_lr(a, i));
        adam1(a, p.y, g.y, m.y, v.y, group_lr(a, i + 1));
        adam1(a, p.z, g.z, m.z, v.z, group_lr(a, i + 2));
        adam1(a, p.w, g.w, m.w, v.w, group_lr(a, i + 3));
        reinterpret_cast<float4 *>(a.p)[q] = p;
        reinterpret_cast<float4 *>(a.m)[q] = m;
        reinterpret_cast<float4 *>(a.v)[q] = v;
    }
    const int64_t tail = 4 * n4 + blockIdx.x * (int64_t)BSR_BLOCK + threadIdx.x;
    if (tail < a.count && tail < 4 * n4 + 4)
        adam1(a, a.p[tail], a.g[tail], a.m[tail], a.v[tail], group_lr(a, tail));
}

__global__ void adam_bump_kernel(int64_t *step) { *step += 1; }

}  // namespace bsr

using namespace bsr;

static int adam_impl(float *params, const float *grads, float *exp_avg, float *exp_avg_sq, int64_t count,
                     int32_t n_groups, const int64_t *group_end, const float *group_lr, int64_t step,
                     int64_t *step_dev, double beta1, double beta2, double eps, void *stream) {
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
    const int64_t n4 = count / 4;
    const unsigned blocks = (unsigned)imax64(1, imin64(div_up(imax64(n4, 1), BSR_BLOCK), 148 * 8));
    adam_kernel<<<blocks, BSR_BLOCK, 0, (cudaStream_t)stream>>>(a);
    if (step_dev) adam_bump_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(step_dev);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_adam_step(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                             int64_t count, int32_t n_groups, const int64_t *group_end,
                             const float *group_lr, int64_t step, double beta1, double beta2,
                             double eps, void *stream) {
    return adam_impl(params, grads, exp_avg, exp_avg_sq, count, n_groups, group_end, group_lr, step, nullptr,
                     beta1, beta2, eps, stream);
}

extern "C" int bsr_adam_step_device(float *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                                    int64_t count, int32_t n_groups, const int64_t *group_end,
                                    const float *group_lr, int64_t *step_counter, double beta1,
                                    double beta2, double eps, void *stream) {
    if (!step_counter) return BSR_ERR_BAD_ARG;
    return adam_impl(params, grads, exp_avg, exp_avg_sq, count, n_groups, group_end, group_lr, 0, step_counter,
                     beta1, beta2, eps, stream);
}
