// Dev microbenchmark: shared-memory LDS.64 throughput on sm_100a and the
// ceiling of the FSE update-loop instruction mix without its argmax chain.
//   mode 0: pure LDS.64 gathers (32 lanes x 8 B, conflict-free, immediate row offsets)
//   mode 1: the update mix per bin (2 LDS.64, 2 FADD2, 2 FFMA2, |g|^2, FMNMX) over 11 bins,
//           no barrier / argmax
//   mode 2: mode 1 plus one __syncthreads per iteration
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldsbw ldsbw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int F = 64, NB = 11, RSTEP = 3, ROWS = 97;

__device__ __forceinline__ unsigned long long f2u(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 u2f(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}

template <int MODE>
__global__ void __launch_bounds__(192, 4) k(float *out, long long *cyc, int iters) {
    extern __shared__ float2 W[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int i = t; i < ROWS * F; i += blockDim.x) W[i] = make_float2(1e-3f * (i & 255), 1e-3f * (i % 91));
    __syncthreads();
    const int u0 = warp / 2, v = (warp & 1) * 32 + lane;
    float2 G[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) G[j] = make_float2(v * 0.01f + j, u0 * 0.02f);
    float tmax = 0.f, gpr = 0.001f, gpi = 0.002f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int a = (it * 7) & 31, b = (it * 13) & 63;
        const int cm = (v - b) & (F - 1), cp = (v + b) & (F - 1);
        const float2 *lo = W + (u0 - a + F / 2) * F + cm;
        const float2 *hi = W + (u0 + a + F / 2) * F + cp;
        if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const float2 x = lo[j * RSTEP * F], y = hi[j * RSTEP * F];
                G[j] = cadd(G[j], cadd(x, y));
            }
        } else {
#pragma unroll
            for (int j0 = 0; j0 < NB; j0 += 4) {
                float2 wl[4], wh[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (j0 + q < NB) {
                        wl[q] = lo[(j0 + q) * RSTEP * F];
                        wh[q] = hi[(j0 + q) * RSTEP * F];
                    }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (j0 + q < NB) {
                        const int j = j0 + q;
                        const float2 S = cadd(wl[q], wh[q]), D = csub(wl[q], wh[q]);
                        G[j] = cfma(make_float2(-gpr, -gpr), S, G[j]);
                        G[j] = cfma(make_float2(D.y, -D.x), make_float2(gpi, gpi), G[j]);
                        tmax = fmaxf(tmax, __fmaf_rn(G[j].x, G[j].x, __fmul_rn(G[j].y, G[j].y)));
                    }
            }
            gpr = tmax * 1e-9f;
            if (MODE == 2) __syncthreads();
        }
    }
    long long t1 = clock64();
    float s = tmax;
#pragma unroll
    for (int j = 0; j < NB; ++j) s += G[j].x + G[j].y;
    out[blockIdx.x * blockDim.x + t] = s;
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = ROWS * F * sizeof(float2) + 3000;
    float *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * 192 * sms * 8);
    cudaMalloc(&cyc, sizeof(long long) * sms * 8);
    const int iters = 4000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int per_sm = 1; per_sm <= 4; per_sm *= 2) {
            auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            const int grid = sms * per_sm;
            fn<<<grid, 192, smem>>>(out, cyc, 10);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            fn<<<grid, 192, smem>>>(out, cyc, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            long long c;
            cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            // bytes of W gathered per SM: windows/SM x iters x 2112 bins x 16 B
            const double bytes = (double)per_sm * iters * 6 * 32 * NB * 16;
            const double flops = (double)grid * iters * 6 * 32 * NB * 17;
            printf("mode %d  ctas/SM %d  cycles/iter/window %.1f  LDS B/clk/SM %.1f  %.1f TFLOP/s-equiv (17/bin) %s\n",
                   mode, per_sm, (double)c / iters, bytes / (double)c, flops / (ms * 1e-3) / 1e12,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
