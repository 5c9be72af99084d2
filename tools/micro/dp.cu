// FP64 pipe numbers on sm_100a: DFMA / DADD latency (dependent chains) and
// throughput of DFMA and of the fp32 <-> fp64 conversions (F2F), per SM per
// clock, one CTA of 1024 threads per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dp tools/micro/dp.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void lat(double *out, long long *cyc, double seed) {
    double v = seed + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) v = fma(v, 1.0000001, 0.5);
    long long t1 = clock64();
    cyc[0] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) v = v + 0.25;
    t1 = clock64();
    cyc[1] = t1 - t0;
    float f = (float)seed;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) f = (float)((double)f * 1.0000001);
    t1 = clock64();
    cyc[2] = t1 - t0;  // F2F.F64.F32 + DMUL + F2F.F32.F64 chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) f = f * 1.0000001f + 0.5f;
    t1 = clock64();
    cyc[3] = t1 - t0;
    out[threadIdx.x] = v + f;
}

// 8 independent accumulators per thread
__global__ void tput_dfma(double *out, double seed) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 1.0000001, 0.5);
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// conversions fp32 -> fp64 (8 independent per thread per step), result folded
// with an integer op so the compiler keeps every conversion
__global__ void tput_f2d(double *out, float seed) {
    float f[8];
    unsigned long long acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = seed + j + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const double d = (double)f[j];
            acc ^= (unsigned long long)__double_as_longlong(d);
            f[j] = __int_as_float(__float_as_int(f[j]) + 1);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (double)acc;
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(double) * 2);
    cudaMalloc(&cyc, 16 * sizeof(long long));
    lat<<<1, 32>>>(out, cyc, 1.0);
    long long h[4];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("latency cycles: DFMA %.1f  DADD %.1f  F2F+DMUL+F2F %.1f  FFMA %.1f\n", h[0] / (double)N, h[1] / (double)N,
           h[2] / (double)N, h[3] / (double)N);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        tput_dfma<<<148, 1024>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 148.0 * 1024 * N * 8;
        if (rep) printf("DFMA: %.2f TFLOP/s = %.1f /clk/SM at %d MHz (nominal clock)\n", 2 * ops / ms / 1e9,
                        ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
        cudaEventRecord(e0);
        tput_f2d<<<148, 1024>>>(out, 1.0f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("F2F.F64.F32 (+2 int ops): %.1f conversions /clk/SM at %d MHz\n", ops / (ms * 1e-3) / 148 / (clk * 1e3),
                        clk / 1000);
    }
    return 0;
}
