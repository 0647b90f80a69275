// Micro-benchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float a, float b) {
    return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

__global__ void k_ffma(float* out, int iters, float s) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    float m = s, c = 0.999f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], m, c);  // 3-register form (m, c in registers)
    }
    float r = 0;
    for (int i = 0; i < 8; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma2(float* out, int iters, float s) {
    unsigned long long a[8];
    for (int i = 0; i < 8; ++i) a[i] = f2(threadIdx.x * 0.001f + i, threadIdx.x * 0.002f + i);
    unsigned long long m = f2(s, s), c = f2(0.999f, 0.999f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], m, c);
    }
    float r = 0;
    for (int i = 0; i < 8; ++i) r += __uint_as_float(unsigned(a[i])) + __uint_as_float(unsigned(a[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float t1, t2;
        cudaEventRecord(e0);
        k_ffma<<<148 * 8, 256>>>(out, iters, 1.0001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t1, e0, e1);
        cudaEventRecord(e0);
        k_ffma2<<<148 * 8, 256>>>(out, iters, 1.0001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t2, e0, e1);
        const double n = 148.0 * 8 * 256 * iters * 8;
        printf("FFMA : %.3f ms, %.1f TFLOP/s\n", t1, 2 * n / t1 / 1e9);
        printf("FFMA2: %.3f ms, %.1f TFLOP/s (2 FMA per instruction)\n", t2, 2 * 2 * n / t2 / 1e9);
    }
    return 0;
}
