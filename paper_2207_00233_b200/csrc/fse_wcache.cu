// Weight-spectrum cache of a device session (sm_100a).
//
// The weight plane of a window (fsefill/fse.py:105-119) is rho^dist from the
// window centre times {1, delta, 0} by sample class, so W = DFT(w)
// (_kernel.pyx:148) depends only on the window's shape (M, N) and its class
// map -- not on image values.  Windows of one session that share both share W
// bit for bit.  On BASELINE config 4 about two thirds of a frame's windows
// share their map with another window of the frame (the interiors of 16x16
// loss areas, seen from blocks in the same relative position and batch order).
//
// Before the first level of a session:
//   1. wsig_kernel     one warp per window: the class map as 2 bits per sample
//                      (row words via ballots), an order-free 64-bit hash of
//                      it, and an insert into an open-addressing table keyed
//                      by the hash (representative = the window that claimed
//                      the slot);
//   2. wassign_kernel  one thread per table slot: maps seen at least twice
//                      (min_count 1: every map) get a plane index, up to the
//                      plane capacity;
//   3. wmatch_kernel   one warp per window: the window's signature is compared
//                      WORD FOR WORD with its representative's, so a hash
//                      collision can only lose a cache hit, never return a
//                      wrong plane; wslot[entry] = plane or -1;
//   4. the MODE 2 launch of the window kernel (fse_inst_fast.cu) computes each
//      plane's half rows from its representative window with the very code
//      the level kernel would run, so cached and computed W are bit-identical.
// The level kernels then read wslot[entry] and, on a hit, skip the w half of
// the column pass, the w row partials and the combine (about 10% of a fp64
// window's time at F = 64) and load the half rows from L2 instead.
#include <cstdint>
#include <string>

#include "fse_kernel.cuh"
#include "fse_wcache.h"

namespace fse {

__device__ __forceinline__ unsigned long long wc_mix(unsigned long long x) {
    // splitmix64 finaliser
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

constexpr int kSigWarps = 8;  // windows per CTA of the per-window kernels

static __global__ void __launch_bounds__(kSigWarps * 32) wsig_kernel(const WCacheArgs A) {
    const int lane = threadIdx.x & 31;
    const int e = blockIdx.x * kSigWarps + (threadIdx.x >> 5);
    if (e >= A.n_entries) return;
    const int2 en = A.entries[e];
    const FrameDesc *fd = A.frames + en.x;
    const int blk = en.y;
    // window geometry (grid.py:108-135), as in the window kernel
    const int r = blk / A.cols, c = blk - r * A.cols;
    const int r0 = r * A.B, c0 = c * A.B;
    const int r1 = min(r0 + A.B, A.H), c1 = min(c0 + A.B, A.W);
    const int wr0 = max(0, r0 - A.d), wc0 = max(0, c0 - A.d);
    const int M = min(A.H, r1 + A.d) - wr0, N = min(A.W, c1 + A.d) - wc0;
    const uint8_t *msk = fd->mask;
    const int32_t *rnk = fd->rank;
    const int myrank = rnk[blk];
    unsigned long long *sg = A.sig + (size_t)e * A.SW;
    const unsigned long long head = ((unsigned long long)M << 32) | (unsigned)N;
    // The kernel is instruction-bound (about 2.5 k warp instructions per
    // 32 x 32 window), so: word w of the signature is kept by lane w % 32 and
    // mixed into the hash once there (not by all 32 lanes), the block row of a
    // sample row is stepped instead of divided, and 8 rows' loads are in
    // flight before their ballots.
    unsigned long long h = 0;  // per-lane partial: order-free sum of per-word mixes
    unsigned long long mine = 0;
    int w = 0;
    constexpr int RB = 8;
    const int by0 = wr0 / A.B, ry0 = wr0 - by0 * A.B;
    auto flush = [&](int wlast) {
        // lanes 0 .. wlast % 32 hold words (wlast & ~31) + lane
        if (lane <= (wlast & 31)) {
            const int k = (wlast & ~31) + lane;
            sg[1 + k] = mine;
            h += wc_mix(mine + (unsigned long long)(k + 1) * 0x9E3779B97F4A7C15ull);
        }
    };
    for (int jc = 0; jc < N; jc += 32) {
        const int j = jc + lane;
        const bool jin = j < N;
        const int x = wc0 + (jin ? j : 0);
        const int bx = x / A.B;
        const uint8_t *mcol = msk + (size_t)wr0 * A.W + x;
        int by = by0, ry = ry0;
        for (int i0 = 0; i0 < M; i0 += RB) {
            uint8_t s[RB];
            int owner[RB], orank[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                const int i = i0 + q;
                s[q] = 0;
                owner[q] = by * A.cols + bx;
                if (jin && i < M) s[q] = mcol[(size_t)i * A.W];
                if (++ry == A.B) {
                    ry = 0;
                    ++by;
                }
            }
#pragma unroll
            for (int q = 0; q < RB; ++q) orank[q] = s[q] == FSE_LOST ? rnk[owner[q]] : 0;
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                const int i = i0 + q;
                if (i >= M) break;  // uniform
                // class: 2 = available (weight rho^dist), 1 = reconstructed
                // (delta rho^dist: written by an earlier batch, or already
                // RECONSTRUCTED in the input mask), 0 = weight 0 (lost and not
                // yet written, or outside the window's columns)
                unsigned cls = 0;
                if (jin) {
                    if (s[q] == FSE_LOST) cls = (owner[q] != blk && orank[q] < myrank) ? 1u : 0u;
                    else cls = s[q] == FSE_RECONSTRUCTED ? 1u : 2u;
                }
                const unsigned b0 = __ballot_sync(0xffffffffu, cls & 1u);
                const unsigned b1 = __ballot_sync(0xffffffffu, cls >> 1);
                if (lane == (w & 31)) mine = ((unsigned long long)b1 << 32) | b0;
                if ((w & 31) == 31) flush(w);
                ++w;
            }
        }
    }
    if (w & 31) flush(w - 1);
    // warp sum of the partial hashes
    {
        unsigned lo = (unsigned)h, hi = (unsigned)(h >> 32);
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const unsigned long long o =
                ((unsigned long long)__shfl_xor_sync(0xffffffffu, hi, off) << 32) | __shfl_xor_sync(0xffffffffu, lo, off);
            h += o;
            lo = (unsigned)h;
            hi = (unsigned)(h >> 32);
        }
        h += wc_mix(head);
    }
    if (lane == 0) {
        sg[0] = head;
        if (h == 0) h = 1;  // 0 marks an empty slot
        // Popular maps are hit by tens of thousands of windows, and atomics on
        // one address serialise in L2 (a CAS + min + add per window made this
        // kernel 3x slower).  So: a plain load first; only a window that finds
        // the slot empty tries the CAS, and the CAS winner is the map's
        // representative (any window of the map serves); a window that finds
        // its hash already there marks the map as shared with a plain store.
        unsigned slot = (unsigned)(h >> 17) & A.tmask;
        for (;;) {
            unsigned long long k = *reinterpret_cast<volatile unsigned long long *>(A.keys + slot);
            if (k == 0ull) {
                k = atomicCAS(A.keys + slot, 0ull, h);
                if (k == 0ull) {
                    A.rep[slot] = (unsigned)e;
                    break;
                }
            }
            if (k == h) {
                A.cnt[slot] = 1u;
                break;
            }
            slot = (slot + 1) & A.tmask;
        }
        A.slot_of[e] = (int)slot;
    }
}

static __global__ void wassign_kernel(const WCacheArgs A) {
    const unsigned n = A.tmask + 1;
    for (unsigned slot = blockIdx.x * blockDim.x + threadIdx.x; slot < n; slot += gridDim.x * blockDim.x) {
        int plane = -1;
        if (A.keys[slot] != 0ull && (A.cnt[slot] != 0u || A.min_count <= 1)) {
            plane = atomicAdd(A.counters, 1);
            if (plane >= A.cap) plane = -1;
            else A.wrep[plane] = (int)A.rep[slot];
        }
        A.cidx[slot] = plane;
    }
}

static __global__ void __launch_bounds__(kSigWarps * 32) wmatch_kernel(const WCacheArgs A) {
    const int lane = threadIdx.x & 31;
    const int e = blockIdx.x * kSigWarps + (threadIdx.x >> 5);
    __shared__ int hits;
    if (threadIdx.x == 0) hits = 0;
    __syncthreads();
    if (e < A.n_entries) {
        const int slot = A.slot_of[e];
        int plane = A.cidx[slot];
        if (plane >= 0) {
            const unsigned rep = A.rep[slot];
            if (rep != (unsigned)e) {
                const unsigned long long *a = A.sig + (size_t)e * A.SW, *b = A.sig + (size_t)rep * A.SW;
                const unsigned long long head = a[0];
                bool same = head == b[0];
                // words in use: rows x 32-column segments of this window
                const int words = 1 + (int)(head >> 32) * (((int)(unsigned)head + 31) >> 5);
                for (int k = 1 + lane; same && k < words; k += 32) same = a[k] == b[k];
                if (!__all_sync(0xffffffffu, same)) plane = -1;
            }
        }
        if (lane == 0) {
            A.wslot[e] = plane;
            if (plane >= 0) atomicAdd(&hits, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && hits) atomicAdd(A.counters + 1, hits);
}

int wcache_classify(const WCacheArgs &a, cudaStream_t s) {
    if (a.n_entries <= 0) return FSE_OK;
    const int grid = (a.n_entries + kSigWarps - 1) / kSigWarps;
    wsig_kernel<<<grid, kSigWarps * 32, 0, s>>>(a);
    FSE_CUDA_TRY(cudaGetLastError());
    const unsigned slots = a.tmask + 1;
    wassign_kernel<<<(int)std::min<unsigned>((slots + 255) / 256, 148u * 16u), 256, 0, s>>>(a);
    FSE_CUDA_TRY(cudaGetLastError());
    wmatch_kernel<<<grid, kSigWarps * 32, 0, s>>>(a);
    FSE_CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(3, std::memory_order_relaxed);
    return FSE_OK;
}

}  // namespace fse
