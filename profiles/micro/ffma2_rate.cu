// Micro-benchmark: issue/throughput of FFMA vs packed FFMA2 (fma.rn.f32x2) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_rate.cu -o ffma2_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long *>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2 *>(&v); }

template <int ILP>
__global__ void ffma1(float *out, float a, float b, int iters) {
    float x[2 * ILP];
#pragma unroll
    for (int i = 0; i < 2 * ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 2 * ILP; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 2 * ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void ffma2(float *out, float a, float b, int iters) {
    unsigned long long x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = f2u(make_float2(threadIdx.x + 2 * i, threadIdx.x + 2 * i + 1));
    const unsigned long long A = f2u(make_float2(a, a)), B = f2u(make_float2(b, b));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) { float2 v = u2f(x[i]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float ms1, ms2;
        cudaEventRecord(e0);
        ffma1<8><<<148 * 8, 256>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms1, e0, e1);
        cudaEventRecord(e0);
        ffma2<8><<<148 * 8, 256>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms2, e0, e1);
        const double fma = 148.0 * 8 * 256 * 16 * (double)iters;
        printf("FFMA : %.3f ms  %.1f TFLOP/s\nFFMA2: %.3f ms  %.1f TFLOP/s\n", ms1, 2 * fma / ms1 / 1e9, ms2,
               2 * fma / ms2 / 1e9);
    }
    return 0;
}
