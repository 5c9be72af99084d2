// Weight-spectrum cache of a device session: see fse_wcache.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fse {

struct FrameDesc;

struct WCacheArgs {
    const FrameDesc *frames;
    const int2 *entries;        // all entries of the session
    int n_entries;
    int H, W, B, d, rows, cols;
    int SW;                     // signature stride in 64-bit words: 1 + Mmax * ceil(Nmax / 32)
    unsigned long long *sig;    // [n_entries][SW]
    unsigned long long *keys;   // hash table (zeroed): key, representative entry, count, plane
    uint32_t *rep;              // (0xFF-filled) the entry that claimed the slot
    uint32_t *cnt;              // (zeroed) 1 = the map was seen again after the claim
    int32_t *cidx;
    uint32_t tmask;             // table slots - 1 (power of two)
    int32_t *slot_of;           // [n_entries]
    int32_t *wslot;             // [n_entries] out: plane index or -1
    int32_t *wrep;              // [cap] out: representative entry of each plane
    int *counters;              // (zeroed) [0] planes wanted (may exceed cap), [1] cache hits
    int cap;                    // plane capacity
    int min_count;              // 2: only maps shared by >= 2 windows get a plane; 1: every map
};

// Queue the three classification kernels on s.
int wcache_classify(const WCacheArgs &a, cudaStream_t s);

}  // namespace fse
