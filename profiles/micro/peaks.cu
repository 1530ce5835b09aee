// Measured compute peaks of this B200 for the raster rooflines (the FP32 / SFU pipes; the
// raster is not a dense contraction, so tensor cores do not apply):
//   FFMA   fma.rn.f32        scalar FP32 FMA            -> TFLOP/s (2 FLOP per lane-op)
//   FFMA2  fma.rn.f32x2      packed pair FMA            -> TFLOP/s (4 FLOP per lane-op)
//   MUFU   ex2.approx.f32    SFU/XU transcendental      -> Gop/s
//   MUFU   rcp.approx.f32    SFU/XU reciprocal          -> Gop/s
// Independent chains (ILP 8) per thread, 148 x 8 CTAs of 256 threads, best of 5, CUDA
// events; the SM clock is read with NVML by the caller (profiles/micro/run_peaks.py).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 peaks.cu -o peaks && ./peaks
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long *>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2 *>(&v); }

constexpr int ILP = 8;

__global__ void k_ffma(float *out, float a, float b, int iters) {
    float x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(a), "f"(b));
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, float a, float b, int iters) {
    unsigned long long x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = f2u(make_float2(threadIdx.x + 2 * i, threadIdx.x + 2 * i + 1));
    const unsigned long long A = f2u(make_float2(a, a)), B = f2u(make_float2(b, b));
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
        const float2 v = u2f(x[i]);
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
__global__ void k_mufu(float *out, int iters) {
    float x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = 0.5f + 1e-3f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            else asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
        }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    const int blocks = 148 * 8, threads = 256;
    float *out;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double lanes = (double)blocks * threads * ILP;
    auto best = [&](auto launch, int iters) {
        float bestms = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            launch(iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < bestms) bestms = ms;
        }
        return (double)bestms;
    };
    const int it_f = 40000, it_m = 8000;
    const double t_ffma = best([&](int n) { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f, n); }, it_f);
    const double t_ffma2 = best([&](int n) { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f, n); }, it_f);
    const double t_ex2 = best([&](int n) { k_mufu<0><<<blocks, threads>>>(out, n); }, it_m);
    const double t_rcp = best([&](int n) { k_mufu<1><<<blocks, threads>>>(out, n); }, it_m);
    printf("{\"ffma_tflops\": %.3f, \"ffma2_tflops\": %.3f, \"ex2_gops\": %.1f, \"rcp_gops\": %.1f, "
           "\"ms\": [%.3f, %.3f, %.3f, %.3f], \"err\": \"%s\"}\n",
           lanes * it_f * 2.0 / (t_ffma * 1e-3) / 1e12, lanes * it_f * 4.0 / (t_ffma2 * 1e-3) / 1e12,
           lanes * it_m / (t_ex2 * 1e-3) / 1e9, lanes * it_m / (t_rcp * 1e-3) / 1e9, t_ffma, t_ffma2, t_ex2,
           t_rcp, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
