// Dependent-chain latency of fp64 / fp32 ops on one thread (clock64), B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false fp64_latency.cu -o fp64_latency
#include <cstdio>
__global__ void chains(double *out, long long *cyc, double a, double b, float fa, float fb) {
    double x = a;
    float y = fa;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = x * b;
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = x + b;
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) y = y * fb;
    long long t3 = clock64();
    // DMUL -> DSETP -> select chain (the replay recurrence's stop test)
    double z = a;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        const double n = z * b;
        z = (n < 1e-300) ? z : n;
    }
    long long t4 = clock64();
    out[0] = x + z;
    out[1] = y;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
}
int main() {
    double *o;
    long long *c, h[4];
    cudaMalloc(&o, 16);
    cudaMalloc(&c, 32);
    for (int r = 0; r < 2; ++r) chains<<<1, 1>>>(o, c, 1.0, 0.999999, 1.f, 0.9999f);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles per op: DMUL %.1f DADD %.1f FMUL %.1f DMUL+DSETP+SEL %.1f\n", h[0] / 1024.0, h[1] / 1024.0,
           h[2] / 1024.0, h[3] / 1024.0);
    return 0;
}
