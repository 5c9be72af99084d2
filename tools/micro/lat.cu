// Latency of warp primitives on sm_100a: dependent chains timed with clock64.
#include <cstdio>
#include <cuda_runtime.h>

#define N 256

__global__ void k(unsigned *out, long long *cyc, unsigned seed) {
    unsigned v = threadIdx.x * seed + 1;
    long long t0, t1;
    const int lane = threadIdx.x & 31;
    // 1. REDUX.MAX chain (result fed back)
    __syncwarp();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) v = __reduce_max_sync(0xffffffffu, v + lane) ;
    t1 = clock64();
    cyc[0] = t1 - t0;
    // 2. SHFL chain
    __syncwarp();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v + 1, 1);
    t1 = clock64();
    cyc[1] = t1 - t0;
    // 3. ballot chain
    __syncwarp();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) v = __ballot_sync(0xffffffffu, (v >> (lane & 7)) & 1) + lane;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // 4. integer add chain (loop overhead baseline)
    __syncwarp();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) v = v * 3 + lane;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // 5. __syncthreads chain (single CTA of this block size)
    __syncthreads();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { __syncthreads(); v += lane; }
    t1 = clock64();
    cyc[4] = t1 - t0;
    // 6. smem store -> barrier -> load chain
    __shared__ unsigned s[32];
    __syncthreads();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        if (lane == 0) s[threadIdx.x >> 5] = v;
        __syncthreads();
        v = s[(v & 1)] + lane;
    }
    t1 = clock64();
    cyc[5] = t1 - t0;
    // 7. REDUX max + min pair (stage-1 argmax shape)
    __syncwarp();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        unsigned m = __reduce_max_sync(0xffffffffu, v);
        unsigned l = __reduce_min_sync(0xffffffffu, v == m ? lane : 99u);
        v = v + l + lane;
    }
    t1 = clock64();
    cyc[6] = t1 - t0;
    // 8. max + ballot (single-winner shape)
    __syncwarp();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        unsigned m = __reduce_max_sync(0xffffffffu, v);
        unsigned b = __ballot_sync(0xffffffffu, v == m);
        v = v + (__ffs(b) - 1) + lane;
    }
    t1 = clock64();
    cyc[7] = t1 - t0;
    out[threadIdx.x] = v;
}

int main() {
    unsigned *o; long long *c, h[8];
    cudaMalloc(&o, 1024 * 4); cudaMalloc(&c, 8 * 8);
    const char *names[8] = {"REDUX.MAX dep", "SHFL dep", "VOTE dep", "IMAD dep", "BAR (192 thr)", "STS+BAR+LDS", "REDUX max+min", "REDUX max+ballot"};
    for (int nt : {32, 192}) {
        k<<<1, nt>>>(o, c, 7);
        k<<<1, nt>>>(o, c, 7);
        cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
        printf("threads %d\n", nt);
        for (int i = 0; i < 8; ++i) printf("  %-18s %6.1f cycles/iter\n", names[i], (double)h[i] / N);
    }
    return 0;
}
