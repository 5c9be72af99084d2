// Fast-path FSE window kernel for square power-of-two DFT sizes F = 32 / 64
// (BASELINE's "FFT 32x32 / 64x64"), sm_100a.  One CTA owns one window.
//
// Reference algorithm: fsefill._kernel.run_fse / _iterate
// (/root/reference/pkg/src/fsefill/_kernel.pyx:14-187), see fse_fit.cuh.
//
// What differs from the generic kernel (fse_kernel.cuh), all for the
// iteration loop's instruction count:
//   * Canonical half spectrum.  Only one bin of every conjugate pair is kept:
//     rows 1..F/2-1 whole, rows 0 and F/2 for v <= F/2.  That is exactly the
//     set of canonical picks (reference tests/reference.py:59-71), and a pick
//     and its twin produce the same update and coefficients, so nothing is
//     lost; ties resolve to the smallest row-major index as in the reference's
//     strict-'>' scan (_kernel.pyx:32-44).
//   * Row-extended weight spectrum.  W is stored for rows -F/2 .. F (3F/2+1
//     rows, W[r] = W[r mod F]); since picks have a <= F/2 and owned rows
//     u <= F/2, both shifted rows u-a and u+a fall inside without a modulo,
//     and a warp's successive rows are a compile-time stride apart, so each
//     gather is one LDS.64/LDS.128 with an immediate offset.
//   * Self-conjugate picks reuse the general update with p halved and made
//     real: (p/2)(W[k-j] + W[k+j]) with W[k-j] = W[k+j]; x2 and /2 are exact.
//   * fp32 near-tie guard.  fp32 rounding moves |g|^2 by up to ~1e-4 of the
//     current maximum after 100 iterations, which can swap two candidates the
//     fp64 reference separates by less than that.  Every iteration the CTA
//     reduces the top-2 energies; when the runner-up is within tau of the
//     winner the window is handed to the fp64 kernel (redo list) and the CTA
//     stops.  The fp64 redo runs before the next level, so results are those
//     of the fp64 path for every guarded window.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include "fse_kernel.cuh"

namespace fse {

// dev instrumentation (-DFSE_CLOCKS): CTA 0, thread 0 records clock64() at the
// phase boundaries of its window (fse_debug_clocks reads them back)
#ifdef FSE_CLOCKS
static __device__ long long g_fse_clk[1024 + 8];
#define FSE_CLK(i)                                                               \
    do {                                                                         \
        if (blockIdx.x == 0 && threadIdx.x == 0 && (i) < 1024 + 8) g_fse_clk[(i)] = clock64(); \
    } while (0)
#else
#define FSE_CLK(i) \
    do {           \
    } while (0)
#endif

template <typename T_, int F_, int NW_, int EXT_ = 1, int MINB_ = 0, int CL_ = 1, bool TRACK_ = false,
          int LG_ = 0>
struct FastCfg {
    // W gathers of LG bins are issued before their math (0 = the build
    // default: FSE_LG32 / FSE_LG64); the narrow-level variants, one CTA per SM
    // with registers to spare, issue all of a thread's gathers at once
    static constexpr int LGC = LG_;
    // TRACK (fp32): every thread carries its best bin (index, g) through the
    // update and the argmax takes one barrier; otherwise fp32 uses the lazy
    // argmax (running maximum only, candidate warps re-find their bin after a
    // second barrier).  Lazy is faster on wide levels (issue-bound), tracked on
    // levels narrower than a few waves (latency-bound).
    static constexpr bool TRACK = TRACK_;
    static constexpr int MINB = MINB_;  // __launch_bounds__ min blocks per SM (0 = unspecified)
    // CL > 1: one window is split over a thread-block cluster of CL CTAs (one
    // per SM): the bins are spread over CL * NW warps, every CTA keeps a full
    // copy of W, and the per-iteration argmax slots are exchanged through DSMEM
    // with one cluster barrier.  For dependency levels narrower than the GPU,
    // where a window's latency, not the throughput, sets the time.
    static constexpr int CL = CL_;
    static constexpr int NWT = NW_ * CL_;       // warps per window
    // EXT: row-extended W (rows -F/2..F, no modulo on the gathers).  !EXT: the
    // plain F-row plane with a per-bin wrap select (2/3 of the shared memory;
    // used where the extended plane would cost occupancy, i.e. fp64 at F = 64).
    static constexpr bool EXT = EXT_ == 1;
    // HALF (EXT_ = 2): only the half rows 0..F/2 of W are stored; rows outside
    // them are read as conj W[-r][-c] (fp64 at F = 128, where even the plain
    // plane, 129 x 128 x 16 B, exceeds shared memory).  The w-combine writes
    // W over the row partials, which share its index map.
    static constexpr bool HALF = EXT_ == 2;
    using T = T_;
    using T2 = typename V2<T_>::type;
    static constexpr int F = F_;
    static constexpr int NW = NW_;
    static constexpr int NT = NW_ * 32;
    static constexpr int R1 = F_ / 2 + 1;       // half-plane rows
    static constexpr int SEG = F_ / 32;         // 32-column segments per row
    static constexpr int NSEGS = R1 * SEG;      // row segments of the half plane
    static constexpr int NB = (NSEGS + NWT - 1) / NWT;  // segments (bins) per thread
    static constexpr int RSTEP = NWT / SEG;     // row stride between a warp's segments
    static constexpr int EXT_ROWS = 3 * F_ / 2 + 1;
    // threads summing the block model (see the write-back): the smallest
    // CTA of any variant of this F
    static constexpr int NSUB_BASE = F_ == 32 ? 96 : F_ == 64 ? 192 : 640;
    static_assert(NW_ * 32 >= NSUB_BASE, "model subsets need NSUB_BASE threads");
    static_assert(F_ == 32 || F_ == 64 || F_ == 128, "fast path: F = 32, 64 or 128");
    static_assert(NW_ % SEG == 0, "NW must be a multiple of F/32");
    static_assert(NWT <= 32, "one warp reduces the window's slots");
    static_assert(NB <= 32, "5-bit bin tag");
};

template <typename T>
struct FastSlot {
    unsigned long long key;  // fp64: exact key; fp32: (energy key << 32) | ~lin
    unsigned int second;     // fp32 guard: energy key of the warp's runner-up
    unsigned int lin;        // row-major index of the warp's best bin
    T gre, gim;              // g of the warp's best bin
};

// A warp's argmax candidate (exact energy key, row-major bin index, g); one
// 16-byte store for fp32.
template <typename T>
struct ArgSlot;
template <>
struct __align__(16) ArgSlot<float> {
    unsigned key, lin;
    float gre, gim;
};
template <>
struct __align__(16) ArgSlot<double> {
    unsigned long long key;
    unsigned lin, pad;
    double gre, gim;
};
static_assert(sizeof(ArgSlot<double>) <= sizeof(FastSlot<double>), "slot region");

// One iteration's contribution to the block model: pick (a, b) and gamma*p.
template <typename T>
struct __align__(16) PickRec {
    int a, b;
    T gpr, gpi;
};

struct FastLayout {
    size_t tw, slots, red, hist, big, yx, yw, xs, ws, part, total;
};

template <typename T>
__host__ __device__ inline FastLayout fast_layout(int F, int NW, int Mmax, int Nmax, int model_n,
                                                  int iters, int ext = 1) {
    FastLayout L;
    const size_t c2 = 2 * sizeof(T);
    size_t o = 0;
    L.tw = o; o += (size_t)F * c2;
    o = (o + 15) & ~size_t(15);
    L.slots = o; o += 2 * (size_t)NW * sizeof(FastSlot<double>);
    L.red = o; o += (size_t)(NW + 2) * sizeof(double);
    o = (o + 15) & ~size_t(15);
    L.hist = o; o += (size_t)(model_n > 0 ? (iters > 0 ? iters : 1) : 1) * sizeof(PickRec<T>);
    o = (o + 127) & ~size_t(127);
    L.big = o;
    const size_t R1 = F / 2 + 1;
    const size_t HS = (size_t)(F / 2) * F * c2;       // ext row F/2 = W row 0
    const size_t HE = (size_t)(F + 1) * F * c2;       // end of ext row F = W row F/2
    const size_t EXT = (size_t)(3 * F / 2 + 1) * F * c2;
    const size_t yb = (R1 * Nmax * c2 + 15) & ~size_t(15);
    const size_t xb = ((size_t)Mmax * Nmax * sizeof(T) + 15) & ~size_t(15);
    const size_t pb = (R1 * (size_t)F * c2 + 15) & ~size_t(15);
    // Phases (each separated by a barrier): column pass reads xs/ws, writes
    // Yx/Yw; row partials read Yx (then Yw) and write part; the x combine reads
    // part into registers, the w combine writes the W half rows [HS, HE) (Yx,
    // Yw, xs, ws dead by then); the extension rows come last.
    L.yx = 0;
    L.yw = yb;
    L.xs = 2 * yb;
    L.ws = L.xs + xb;
    size_t bigb;
    if (ext == 2) {
        // half plane: part (= W after the w-combine, same index map) first,
        // then Yx, Yw; the staging tiles xs / ws live in part's bytes (dead
        // once the column pass has read them, before the first partials)
        L.part = 0;
        L.yx = pb;
        L.yw = pb + yb;
        L.xs = 0;
        L.ws = xb;
        bigb = pb + 2 * yb;
        if (bigb < 2 * xb) bigb = 2 * xb;
    } else if (ext) {
        // partials live above the W half-plane rows [HS, HE), so the w-plane
        // combine can store W rows directly
        L.part = (2 * yb + 2 * xb > HE) ? 2 * yb + 2 * xb : HE;
        bigb = L.part + pb;
        if (bigb < EXT) bigb = EXT;
    } else {
        // plain plane: half rows 0..F/2 at [0, HEc); partials above both the
        // Y planes (read by the partials) and the half rows (written by the
        // w combine); xs / ws are dead once the partials start
        const size_t HEc = (size_t)(F / 2 + 1) * F * c2, FULL = (size_t)(F + 1) * F * c2;
        L.part = 2 * yb > HEc ? 2 * yb : HEc;
        bigb = L.part + pb;
        if (bigb < L.ws + xb) bigb = L.ws + xb;
        if (bigb < FULL) bigb = FULL;
    }
    (void)HS;
    (void)HE;
    L.total = L.big + bigb;
    return L;
}

// Arguments of the fast kernel.
struct FastArgs {
    // MODE 0: pipeline level
    const FrameDesc *frames;
    const int2 *entries;
    int H, W, B, d, rows, cols;
    double delta;
    const double *decay;
    int decay_dim;
    // MODE 1: window operator
    const void *values, *weights;
    void *plog;
    int M, N;
    // both
    int iterations;
    double gamma;
    int32_t *picks;
    // fp32 near-tie guard (MODE 0): redo list for the fp64 kernel
    int2 *redo_list;
    int *redo_count;
    float tau0, tau1;  // guard when e1 - e2 <= (tau0 + tau1 * it) * e1
    // persistent (redo) launch: entries[0 .. *count)
    const int *count;
    // persistent dataflow launch (fse_fast_dataflow_kernel): entries[0 .. total)
    // in dependency-level order, a work counter, one completion flag per
    // (frame, block), and the dependency radius in blocks
    int total;
    int *next;   // [0] queue head, [1] queue tail
    int *done;   // per (frame, block): outstanding dependency count
    int *queue;  // ready queue, total slots, -1 = not yet written
    int R;
    // fused halo exchange (row-band shards over peer memory, MODE 0): the
    // write-back also stores into the upper / lower neighbour's frame (the
    // same coordinates, mapped through CUDA IPC) for blocks whose block row is
    // < peer_up_end / >= peer_down_begin -- the rows the neighbour's windows
    // read.  nullptr = no neighbour on that side.
    void *peer_up, *peer_down;
    int peer_up_end, peer_down_begin;
    // weight-spectrum cache (fse_wcache.cu): W = DFT(w) depends only on a
    // window's shape and class map, not on image values, so windows of one
    // session that share both share W.  wslot[entry] = plane index or -1;
    // wplanes = planes of R1 x F complex (the half rows 0..F/2), written by
    // the MODE 2 launch (one CTA per plane: entry wrep[plane] of `entries`,
    // planes [0, *count)) before the first level.
    const int32_t *wslot;
    void *wplanes;
    const int32_t *wrep;
};

__device__ __forceinline__ unsigned warp_max_u32(unsigned v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ unsigned warp_min_u32(unsigned v) { return __reduce_min_sync(0xffffffffu, v); }

// Keys of non-negative energies for integer REDUX: the IEEE bits of a value
// >= 0 order like the value.
__device__ __forceinline__ unsigned energy_key(float e) { return __float_as_uint(e); }
__device__ __forceinline__ unsigned long long energy_key(double e) {
    return (unsigned long long)__double_as_longlong(e);
}

// |g|^2 with one pinned rounding sequence (y*y, then fma(x, x, .)), so the
// value found again by the winner search equals the one maximised
__device__ __forceinline__ float energy(float2 g) { return __fmaf_rn(g.x, g.x, __fmul_rn(g.y, g.y)); }
__device__ __forceinline__ double energy(double2 g) { return __fma_rn(g.x, g.x, __dmul_rn(g.y, g.y)); }

__device__ __forceinline__ unsigned warp_max_k(unsigned k) { return warp_max_u32(k); }
__device__ __forceinline__ unsigned long long warp_max_k(unsigned long long k) {
    const unsigned mh = warp_max_u32((unsigned)(k >> 32));
    const unsigned ml = warp_max_u32((unsigned)(k >> 32) == mh ? (unsigned)k : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// Warp argmax of (key, lin): largest key, ties to the smallest lin (the
// reference's first maximum in row-major order, _kernel.pyx:32-44).  Returns
// the winning key and lin, uniform across the warp.
__device__ __forceinline__ void warp_argmax(unsigned key, unsigned lin, unsigned &wkey, unsigned &wlin) {
    wkey = warp_max_u32(key);
    wlin = warp_min_u32(key == wkey ? lin : 0xFFFFFFFFu);
}
__device__ __forceinline__ void warp_argmax(unsigned long long key, unsigned lin, unsigned long long &wkey,
                                            unsigned &wlin) {
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = warp_max_u32(hi);
    const unsigned ml = warp_max_u32(hi == mh ? lo : 0u);
    wkey = ((unsigned long long)mh << 32) | ml;
    wlin = warp_min_u32(hi == mh && lo == ml ? lin : 0xFFFFFFFFu);
}

// Warp argmax of (key, lin) as above, returning the lane that holds it (the
// lowest lane among equals) instead of the key: the common case -- one lane
// holds the largest key, or for 64-bit keys the largest high word -- costs one
// REDUX and one ballot; only ties in that first REDUX take the full
// (key, lin) reduction.  Keys are per-lane best-of-bins with strict '>' in
// row-major bin order, so a unique holder's lin is already the first maximum.
__device__ __forceinline__ int warp_argmax_lane(unsigned key, unsigned lin) {
    const unsigned mk = warp_max_u32(key);
    unsigned cand = __ballot_sync(0xffffffffu, key == mk);
    if (__popc(cand) > 1) {
        const unsigned ml = warp_min_u32(key == mk ? lin : 0xFFFFFFFFu);
        cand = __ballot_sync(0xffffffffu, key == mk && lin == ml);
    }
    return __ffs(cand) - 1;
}
__device__ __forceinline__ int warp_argmax_lane(unsigned long long key, unsigned lin) {
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = warp_max_u32(hi);
    unsigned cand = __ballot_sync(0xffffffffu, hi == mh);
    if (__popc(cand) > 1) {
        const unsigned ml = warp_max_u32(hi == mh ? lo : 0u);
        const unsigned mi = warp_min_u32(hi == mh && lo == ml ? lin : 0xFFFFFFFFu);
        cand = __ballot_sync(0xffffffffu, hi == mh && lo == ml && lin == mi);
    }
    return __ffs(cand) - 1;
}

// ---- complex pair arithmetic.  fp32 uses the sm_100 packed f32x2 pipe
// (FADD2 / FFMA2: two lanes of fp32 math per instruction, with scalar
// broadcast and half-swizzle operands), halving the issue slots of the
// update; fp64 is plain scalar math in the same operation order.
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
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return double2{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return double2{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return double2{fma(a.x, b.x, c.x), fma(a.y, b.y, c.y)};
}

// g -= gamma*(p W[k-j] + conj(p) W[k+j]) with gp = gamma*p  (_kernel.pyx:84-91):
//   re: g.x - gpr (lo.x + hi.x) + gpi (lo.y - hi.y)
//   im: g.y - gpr (lo.y + hi.y) - gpi (lo.x - hi.x)
// mS = (-gpr, -gpr), qv = (gpi, -gpi): hoisted out of the bin loop so the
// pairs stay in registers (FFMA2 operands) instead of being rebuilt per bin.
template <typename T2>
__device__ __forceinline__ T2 spectral_update(T2 g, T2 lo, T2 hi, T2 mS, T2 qv) {
    const T2 S = cadd(lo, hi), D = csub(lo, hi);
    g = cfma(mS, S, g);
    return cfma(qv, T2{D.y, D.x}, g);
}

// fp32 form with both FFMA2 multipliers as scalar broadcasts (-gpr, gpi): the
// sign of the imaginary term moves onto the swizzled difference operand
__device__ __forceinline__ float2 spectral_update_bc(float2 g, float2 lo, float2 hi, float ngpr, float gpi) {
    const float2 S = cadd(lo, hi), D = csub(lo, hi);
    g = cfma(float2{ngpr, ngpr}, S, g);
    return cfma(float2{D.y, -D.x}, float2{gpi, gpi}, g);
}

// a / b from the correctly rounded reciprocal rb = 1/b: q = a rb, then one
// FMA residual correction, q + (a - q b) rb, which is the correctly rounded
// quotient for normal operands (Markstein) -- the result of a / b, at 3
// DFMA-pipe operations instead of a full division per use
__device__ __forceinline__ double div_by(double a, double b, double rb) {
    const double q = a * rb;
    return fma(fma(-q, b, a), rb, q);
}

// acc += z * e^{-j theta}, tw = (cos theta, sin theta): the forward-DFT MAC
template <typename T2>
__device__ __forceinline__ T2 dft_mac(T2 acc, T2 z, T2 tw) {
    acc = cfma(z, T2{tw.x, tw.x}, acc);
    return cfma(T2{z.y, -z.x}, T2{tw.y, tw.y}, acc);
}

// WC: this window's W half rows are read from the session's cache plane `wc`
// instead of being computed.  A compile-time flag, so the computing path keeps
// exactly the code (and ptxas schedule) it has without the cache: a run-time
// flag through the set-up cost the fp64 kernel 3.5% on config 4.
template <class C, int MODE, bool GUARD, typename IT, bool WC = false>
__device__ __forceinline__ void fast_window(const FastArgs &A, const FastLayout &L, const int entry_idx,
                                            unsigned char *sm, int2 entry_in = make_int2(-1, -1), int wc = -1) {
    using T = typename C::T;
    using T2 = typename C::T2;
    constexpr int F = C::F, NW = C::NW, NT = C::NT, NB = C::NB, R1 = C::R1, SEG = C::SEG;
    constexpr int RSTEP = C::RSTEP, CL = C::CL, NWT = C::NWT;
    constexpr bool IS_F32 = sizeof(T) == 4;
    static_assert(CL == 1 || (MODE == 0 && !GUARD), "clusters: pipeline mode without the guard");
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int crank = 0;  // rank of this CTA in its cluster
    if constexpr (CL > 1) crank = (int)cooperative_groups::this_cluster().block_rank();
    const int gwarp = crank * NW + warp;  // warp index within the window

    T2 *tw = reinterpret_cast<T2 *>(sm + L.tw);
    FastSlot<T> *slots = reinterpret_cast<FastSlot<T> *>(sm + L.slots);
    double *red = reinterpret_cast<double *>(sm + L.red);
    unsigned char *big = sm + L.big;
    T2 *Wext = reinterpret_cast<T2 *>(big);
    T2 *Yx = reinterpret_cast<T2 *>(big + L.yx);
    T2 *Yw = reinterpret_cast<T2 *>(big + L.yw);
    T *xs = reinterpret_cast<T *>(big + L.xs);
    T *ws = reinterpret_cast<T *>(big + L.ws);
    T2 *part = reinterpret_cast<T2 *>(big + L.part);
    PickRec<T> *hist = reinterpret_cast<PickRec<T> *>(sm + L.hist);

    // ---- window geometry (grid.py:108-135)
    int M, N, br0 = 0, bc0 = 0, bh = 0, bw = 0, wr0 = 0, wc0 = 0, frame = 0, blk = 0;
    const FrameDesc *fd = nullptr;
    int2 entry = make_int2(0, 0);
    static_assert(!WC || (MODE == 0 && C::CL == 1), "cached W: pipeline levels, one CTA per window");
    if constexpr (MODE == 2) {
        if (entry_idx >= *A.count) return;  // planes beyond the session's count
        entry = A.entries[A.wrep[entry_idx]];
    }
    if constexpr (MODE == 0) {
        entry = entry_in.x >= 0 ? entry_in : A.entries[entry_idx];
    }
    constexpr bool cached = WC;
    constexpr bool PIPE = MODE == 0 || MODE == 2;  // window from a frame (vs. the operator's arrays)
    if constexpr (PIPE) {
        frame = entry.x;
        blk = entry.y;
        fd = A.frames + frame;
        const int r = blk / A.cols, c = blk - r * A.cols;
        const int r0 = r * A.B, c0 = c * A.B;
        const int r1 = min(r0 + A.B, A.H), c1 = min(c0 + A.B, A.W);
        wr0 = max(0, r0 - A.d);
        wc0 = max(0, c0 - A.d);
        M = min(A.H, r1 + A.d) - wr0;
        N = min(A.W, c1 + A.d) - wc0;
        br0 = r0 - wr0;
        bc0 = c0 - wc0;
        bh = r1 - r0;
        bw = c1 - c0;
    } else {
        M = A.M;
        N = A.N;
    }

    FSE_CLK(0);
    // ---- e^{+j 2 pi k / F}
    for (int k = t; k < F; k += NT) {
        double s, c;
        sincospi(2.0 * k / F, &s, &c);
        tw[k] = T2{(T)c, (T)s};
    }

    // ---- staging: classes -> weights (fse.py:105-119); x = w * select(w > 0, v, 0)
    double wsum = 0.0;
    if constexpr (PIPE) {
        // a warp stages window rows (lane = column: coalesced mask / image
        // reads, no index division); the global loads of RB rows are issued
        // before any of their math so their latencies overlap
        const int myrank = fd->rank[blk];
        const IT *img = reinterpret_cast<const IT *>(fd->image);
        const uint8_t *msk = fd->mask;
        const int32_t *rnk = fd->rank;
        // staged window rows per warp pass (loads issued before their math);
        // measured on config 4: fp32 RB 2/4/6 = 285.5/283.3/286.1 ms, fp64
        // RB 4/6/8 = 554.4/548.5/558.4 ms
#ifndef FSE_RB
#define FSE_RB 4
#endif
#ifndef FSE_RB64
#define FSE_RB64 6
#endif
        constexpr int RB = IS_F32 ? FSE_RB : FSE_RB64;
        for (int jc = 0; jc < N; jc += 32) {
            const int j = jc + lane;
            const bool jin = j < N;
            const int x = wc0 + (jin ? j : 0);
            const int bx = x / A.B;
            const int dj = abs(2 * j - (N - 1));
            for (int i0 = warp; i0 < M; i0 += NW * RB) {
                uint8_t s[RB];
                IT val[RB];
                int32_t orank[RB], owner[RB];
                double dec[RB];
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    const int i = i0 + r * NW;
                    if (jin && i < M) {
                        const int y = wr0 + i;
                        const size_t off = (size_t)y * A.W + x;
                        owner[r] = (y / A.B) * A.cols + bx;
                        s[r] = msk[off];
                        val[r] = img[off];
                        orank[r] = rnk[owner[r]];
                        dec[r] = A.decay[abs(2 * i - (M - 1)) * A.decay_dim + dj];
                    }
                }
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    const int i = i0 + r * NW;
                    if (jin && i < M) {
                        double w;
                        if (s[r] == FSE_LOST) {
                            // R iff the owner block was written by an earlier batch
                            // (snapshot semantics, conceal.py:148-163); BI/BO otherwise
                            w = (owner[r] != blk && orank[r] < myrank) ? A.delta * dec[r] : 0.0;
                        } else if (s[r] == FSE_RECONSTRUCTED) {
                            w = A.delta * dec[r];
                        } else {
                            w = dec[r];
                        }
                        const double v = (double)val[r];
                        xs[i * N + j] = w > 0.0 ? (T)(w * v) : (T)0;
                        if constexpr (!cached) ws[i * N + j] = (T)w;
                        wsum += w;
                    }
                }
            }
        }
    } else {
        const T *val = reinterpret_cast<const T *>(A.values) + (size_t)entry_idx * M * N;
        const T *wgt = reinterpret_cast<const T *>(A.weights) + (size_t)entry_idx * M * N;
        for (int idx = t; idx < M * N; idx += NT) {
            const double w = (double)wgt[idx];
            const double r0 = w > 0.0 ? (double)val[idx] : 0.0;
            xs[idx] = (T)(w * r0);
            ws[idx] = (T)w;
            wsum += w;
        }
    }
    for (int off = 16; off; off >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, off);
    if (lane == 0) red[warp] = wsum;
    __syncthreads();
    FSE_CLK(1);
    double total = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) total += red[w];

    // ---- DFT pass 1 (columns): Y[k1][n] = sum_m x[m][n] e^{-j 2 pi k1 m / F}, k1 <= F/2.
    // x is real, so with even/odd partial sums Ee, Eo over m:
    //   Y[k1] = Ee + Eo,  Y[F/2 - k1] = conj(Ee - Eo)    (e^{-j pi m} = (-1)^m)
    // and only k1 <= F/4 is summed.
    // Lanes take columns n (conflict-free sample reads), warps take k1 = warp +
    // NW r, so one read of x[m][n], w[m][n] feeds KR outputs; the twiddle
    // index is warp-uniform (broadcast read).
    // (DOX / DOW: a cached window skips the w half, the cache's producer
    // launch the x half)
    auto column_pass = [&](auto dox_, auto dow_) {
        constexpr bool DOX = decltype(dox_)::value, DOW = decltype(dow_)::value;
        constexpr int K1N = F / 4 + 1, KR = (K1N + NW - 1) / NW;
        for (int nc = 0; nc < N; nc += 32) {
            const int n = nc + lane;
            if (n < N) {
                T2 Xe[KR], Xo[KR], We[KR], Wo[KR];
                int kk[KR];
#pragma unroll
                for (int r = 0; r < KR; ++r) {
                    Xe[r] = Xo[r] = We[r] = Wo[r] = T2{0, 0};
                    kk[r] = 0;
                }
                for (int m = 0; m < M; m += 2) {
                    T xv = (T)0, wv = (T)0, xu = (T)0, wu = (T)0;
                    if constexpr (DOX) xv = xs[m * N + n];
                    if constexpr (DOW) wv = ws[m * N + n];
                    const bool odd = m + 1 < M;
                    if constexpr (DOX) xu = odd ? xs[(m + 1) * N + n] : (T)0;
                    if constexpr (DOW) wu = odd ? ws[(m + 1) * N + n] : (T)0;
#pragma unroll
                    for (int r = 0; r < KR; ++r) {
                        const int k1 = warp + NW * r;
                        if (k1 < K1N) {
                            const T2 tv = tw[kk[r]];
                            if constexpr (DOX) Xe[r] = cfma(T2{xv, -xv}, tv, Xe[r]);  // x e^{-j theta}
                            if constexpr (DOW) We[r] = cfma(T2{wv, -wv}, tv, We[r]);
                            const T2 tu = tw[(kk[r] + k1) & (F - 1)];
                            if constexpr (DOX) Xo[r] = cfma(T2{xu, -xu}, tu, Xo[r]);
                            if constexpr (DOW) Wo[r] = cfma(T2{wu, -wu}, tu, Wo[r]);
                            kk[r] = (kk[r] + 2 * k1) & (F - 1);
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < KR; ++r) {
                    const int k1 = warp + NW * r;
                    if (k1 < K1N) {
                        if constexpr (DOX) Yx[k1 * N + n] = cadd(Xe[r], Xo[r]);
                        if constexpr (DOW) Yw[k1 * N + n] = cadd(We[r], Wo[r]);
                        if (k1 != F / 4) {
                            if constexpr (DOX) {
                                const T2 dx = csub(Xe[r], Xo[r]);
                                Yx[(F / 2 - k1) * N + n] = T2{dx.x, -dx.y};
                            }
                            if constexpr (DOW) {
                                const T2 dw = csub(We[r], Wo[r]);
                                Yw[(F / 2 - k1) * N + n] = T2{dw.x, -dw.y};
                            }
                        }
                    }
                }
            }
        }
    };
    {
        using Yes = std::true_type;
        using No = std::false_type;
        if constexpr (MODE == 2) column_pass(No{}, Yes{});
        else if constexpr (cached) column_pass(Yes{}, No{});
        else column_pass(Yes{}, Yes{});
    }
    __syncthreads();
    FSE_CLK(2);

    // ---- bin ownership: warp w owns row segments w + NWT*j: row u0 + RSTEP*j,
    // columns seg*32 + lane (w = the warp's index within the window).
    const int seg = gwarp % SEG;
    const int u0 = gwarp / SEG;
    const int v = seg * 32 + lane;

    // ---- DFT pass 2 (rows), radix-4 over the owners of columns v0 + q F/4:
    //   P_r = sum_{n = r mod 4} Y[u][n] e^{-j 2 pi v0 n / F},
    //   G[u][v0 + q F/4] = sum_r (-j)^{q r} P_r.
    // The owner of quarter q computes P_q (N/4 terms) into `part`, then every
    // owner combines the four partials of its bins.  g is kept for canonical
    // bins; W goes to registers first, to the ext rows once `part` is dead.
    constexpr int QW = F / 4;
    const int q4 = v / QW, v0 = v - q4 * QW;
    // the twiddle sequence e^{-j 2 pi v0 n / F}, n = q4 + 4 i, is the same for
    // every row: its first NR terms (n < 4 NR) stay in registers
    // (measured: fp32 NR 4/6/8 = 293.9/293.3/283.3 ms; fp64 NR 4/6/8 = 554/571/583 ms, spills)
#ifndef FSE_NR32
#define FSE_NR32 8
#endif
#ifndef FSE_NR64
#define FSE_NR64 4
#endif
    constexpr int NR = IS_F32 ? FSE_NR32 : FSE_NR64;
    const int tstep = (4 * v0) & (F - 1);
    T2 twr[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) twr[i] = tw[(v0 * q4 + tstep * i) & (F - 1)];
#ifndef FSE_TW_ROT
#define FSE_TW_ROT 1
#endif
    constexpr bool TW_ROT = !IS_F32 && FSE_TW_ROT;
    const T2 trot = tw[tstep];  // e^{+j 2 pi 4 v0 / F}
    auto part_one = [&](const T2 *Y, int j) {
        {
            const int u = u0 + RSTEP * j;
            if (u < R1) {
                const T2 *yr = Y + u * N;
                T2 acc = T2{0, 0};
#pragma unroll
                for (int i = 0; i < NR; ++i)
                    if (q4 + 4 * i < N) acc = dft_mac(acc, yr[q4 + 4 * i], twr[i]);
                if constexpr (TW_ROT) {
                    // fp64: the remaining twiddles by rotation from the last
                    // register one (per-lane table indices conflict in banks:
                    // 8% of the kernel's shared wavefronts, 45% excess)
                    T2 tc = twr[NR - 1];
                    for (int n = q4 + 4 * NR; n < N; n += 4) {
                        tc = T2{fma(tc.x, trot.x, -tc.y * trot.y), fma(tc.x, trot.y, tc.y * trot.x)};
                        acc = dft_mac(acc, yr[n], tc);
                    }
                } else {
                    int k = (v0 * q4 + tstep * NR) & (F - 1);
                    for (int n = q4 + 4 * NR; n < N; n += 4) {
                        acc = dft_mac(acc, yr[n], tw[k]);
                        k = (k + tstep) & (F - 1);
                    }
                }
                part[(u * 4 + q4) * QW + v0] = acc;
            }
        }
    };
    auto partials = [&](const T2 *Y) {
        // (-DFSE_PART_NOUNROLL halves the kernel's code: config 1 fp64 1.9 vs
        // 2.0 ms, but config 4 fp32 +6%, fp64 +0.5%: unrolled by default)
#ifdef FSE_PART_NOUNROLL
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int j = 0; j < NB; ++j) part_one(Y, j);
    };
    // the w pass runs while G is live in registers: rolled, it needs fewer
    // of them (dev knob FSE_W_ROLLED)
    auto partials_w = [&](const T2 *Y) {
#if defined(FSE_W_ROLLED) && FSE_W_ROLLED
#pragma unroll 1
        for (int j = 0; j < NB; ++j) part_one(Y, j);
#else
        partials(Y);
#endif
    };
    auto combine = [&](int u) -> T2 {
        const T2 *pr = part + (u * 4) * QW + v0;
        T2 acc = pr[0];
#pragma unroll
        for (int r = 1; r < 4; ++r) {
            // + pv (-j)^k, k = q r mod 4, branch-free (q differs within a warp):
            // k=0 (x, y), 1 (y, -x), 2 (-x, -y), 3 (-y, x)
            const T2 pv = pr[r * QW];
            const int k = (q4 * r) & 3;
            const T x = (k & 1) ? pv.y : pv.x, y = (k & 1) ? pv.x : pv.y;
            acc = cadd(acc, T2{(k & 2) ? -x : x, (k == 1 || k == 2) ? -y : y});
        }
        return acc;
    };
    T2 G[NB];
    unsigned valid = 0;  // bit j: bin j is a canonical in-range bin
    if constexpr (MODE != 2) {
        partials(Yx);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int u = u0 + RSTEP * j;
            G[j] = T2{0, 0};
            if (u < R1 && !((u == 0 || u == F / 2) && v > F / 2)) {
                G[j] = combine(u);
                valid |= 1u << j;
            }
        }
        __syncthreads();
    }
    FSE_CLK(3);
    if constexpr (!cached) {
        partials_w(Yw);
        __syncthreads();
    }
    FSE_CLK(1000);
    // a cached window's half rows come from the session's W cache (the bits
    // the combine below would produce: the producer is this very code)
    const T2 *wcache = nullptr;
    if constexpr (cached) wcache = reinterpret_cast<const T2 *>(A.wplanes) + (size_t)wc * (R1 * F);
    if constexpr (MODE == 2) {
        // producer: the half rows go to the cache plane and the CTA is done
        T2 *plane = reinterpret_cast<T2 *>(A.wplanes) + (size_t)entry_idx * (R1 * F);
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int u = u0 + RSTEP * j;
            if (u < R1) plane[u * F + v] = combine(u);
        }
        return;
    }
    auto whalf = [&](int u) -> T2 {
        if constexpr (cached) return wcache[u * F + v];
        else return combine(u);
    };
    // W half rows 0..F/2; with EXT (one CTA per window) also the negative
    // rows W[-u][-v] = conj W[u][v] at once: they land in the dead x/w/Y
    // staging bytes below the half rows, while `part` (above them) is still
    // being read by other threads
    constexpr bool MIRROR_NOW = C::EXT && CL == 1;
    if constexpr (C::HALF) {
        // in place over the partials (same index map u F + v): a row's four
        // quarter partials are all read before any of its W entries lands;
        // the rows of one j are disjoint from every other j's
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int u = u0 + RSTEP * j;
            T2 wv = T2{0, 0};
            if (u < R1) wv = whalf(u);
            __syncthreads();
            if (u < R1) Wext[u * F + v] = wv;
        }
    } else {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int u = u0 + RSTEP * j;
            if (u < R1) {
                const T2 wv = whalf(u);
                Wext[(u + (C::EXT ? F / 2 : 0)) * F + v] = wv;
                if (MIRROR_NOW && u >= 1) Wext[(F / 2 - u) * F + ((F - v) & (F - 1))] = T2{wv.x, -wv.y};
            }
        }
    }
    if constexpr (CL > 1) {
        // every CTA of the cluster holds the whole W: fetch the half rows the
        // other CTAs computed (row u belongs to window warp (u % RSTEP) * SEG)
        auto cluster = cooperative_groups::this_cluster();
        cluster.sync();
        for (int idx = t; idx < R1 * F; idx += NT) {
            const int u = idx / F;
            const int owner = ((u % RSTEP) * SEG) / NW;
            if (owner == crank) continue;
            T2 *p = Wext + (u + (C::EXT ? F / 2 : 0)) * F + (idx - u * F);
            *p = *cluster.map_shared_rank(p, owner);
        }
    }
    __syncthreads();
    FSE_CLK(1001);
    if constexpr (!C::EXT && !C::HALF) {
        // plain plane: rows F/2+1 .. F-1 by W[r][c] = conj W[F-r][-c], and
        // row F = row 0 (the update's row u + a <= F then never wraps)
        for (int idx = t; idx < (F / 2) * F; idx += NT) {
            const int rr = F / 2 + 1 + idx / F, c = idx % F;
            const T2 src = Wext[((F - rr) & (F - 1)) * F + (rr == F ? c : (F - c) & (F - 1))];
            Wext[rr * F + c] = rr == F ? src : T2{src.x, -src.y};
        }
    }
    // extension rows: W[-s] = conj W[s] reflected, W[F] = W[0]
    for (int idx = t; C::EXT && !MIRROR_NOW && idx < (F / 2) * F; idx += NT) {
        const int rr = idx / F, c = idx - rr * F;  // ext row rr in [0, F/2): W row rr - F/2
        const int s = F / 2 - rr;                  // W row -s, s in [1, F/2]
        const T2 src = Wext[(s + F / 2) * F + ((F - c) & (F - 1))];
        Wext[rr * F + c] = T2{src.x, -src.y};
    }
    for (int idx = t; C::EXT && idx < (F / 2) * F; idx += NT) {
        const int rr = F + 1 + idx / F, c = idx % F;  // ext row rr in (F, 3F/2]: W row rr - F/2
        const int s = rr - F / 2;                     // in (F/2, F]
        T2 val;
        if (s == F) {
            val = Wext[(F / 2) * F + c];
        } else {
            const T2 src = Wext[(F - s + F / 2) * F + ((F - c) & (F - 1))];
            val = T2{src.x, -src.y};
        }
        Wext[rr * F + c] = val;
    }
    __syncthreads();

    // sum(w) (_kernel.pyx:144): fp64 takes W[0][0] = sum_mn w[m][n] e^0, which
    // the DFT passes form in an order fixed by F and the window alone, so every
    // variant of one F (warps per window, executor) divides by the same bits;
    // the staging sum above depends on the warp count.  fp32 rounds the
    // double staging sum to float.
    double total_used = total;
    if constexpr (!IS_F32) total_used = (double)Wext[C::EXT ? (F / 2) * F : 0].x;
    const T gamma = (T)A.gamma;
    const T tot = (T)total_used;
    const T inv_tot = (T)1 / tot;
    const int I = A.iterations;
    int32_t *picks_out = nullptr;
    T *plog = nullptr;
    if constexpr (MODE == 0) {
        if (A.picks) picks_out = A.picks + ((size_t)frame * A.rows * A.cols + blk) * (size_t)I * 2;
    } else {
        picks_out = A.picks + (size_t)entry_idx * I * 2;
        plog = reinterpret_cast<T *>(A.plog) + (size_t)entry_idx * I * 2;
    }

    // ---- per-thread argmax state over the owned bins
    // fp32 guard: packed 32-bit keys (energy bits with a 5-bit bin tag, larger =
    // better, smaller j wins ties) and the runner-up.  Otherwise the exact
    // energy with the row-major index of its bin.  Energies are >= 0, so their
    // IEEE bits order like the values, and starting from 0 with no bin is the
    // reference's strict-'>' scan from -1 up to its all-zero case (below).
    unsigned k1 = 0, k2 = 0;
    // (two interleaved even/odd running maxima were measured 4% slower: more
    // registers and moves than the serial compare chain costs)
    T best = (T)0;
    unsigned blin = 0xFFFFFFFFu;       // row-major index of the best bin, none yet
    const unsigned lin0 = (unsigned)(u0 * F + v);
    T2 bg = T2{0, 0};  // g of the best bin, carried along (no register indexing later)
    // LAZY: only the running maximum energy is kept per bin (one FMNMX); the
    // few lanes holding the CTA maximum find its bin again after the reduction
    // (a second barrier), instead of every bin carrying index and g along.
    constexpr bool LAZY = IS_F32 && CL == 1 && !GUARD && !C::TRACK;
    T tmax = (T)0;
    using KeyT = decltype(energy_key((T)0));
    // LAZY64 (fp64): the running maximum of the energies' HIGH words only --
    // one integer max per bin instead of a compare and seven moves.  The high
    // word of a double >= 0 orders like the value to 20 mantissa bits, so the
    // CTA maximum H of the high words selects the candidate bins (high word
    // == H, i.e. within ~1e-6 relative of the maximum); the lanes holding
    // them recompute those energies exactly and resolve the argmax on the full
    // 64-bit keys, ties to the smallest row-major index, after a second
    // barrier -- the same first maximum as the strict '>' scan of
    // _kernel.pyx:32-44.  (Non-finite energies, i.e. NaN/inf inputs, and
    // energies below 2^-1002 are outside this contract.)
    // Measured slower than the tracked one-barrier argmax (config 4 fp64
    // 564.6 vs 545.5 ms, config 1 2.1 vs 1.9 ms: the second barrier costs more
    // than the moves it saves), so opt-in only (-DFSE_LAZY64).
#ifdef FSE_LAZY64
    constexpr bool LAZY64 = !IS_F32 && CL == 1 && !GUARD && !C::TRACK;
#else
    constexpr bool LAZY64 = false;
#endif
    unsigned hmax = 0;
    auto track = [&](int j, T e) {
        if constexpr (LAZY64) {
            hmax = max(hmax, (unsigned)__double2hiint((double)e));
        } else if constexpr (LAZY) {
            tmax = fmax(tmax, e);  // NaN never wins, like the strict '>' scan
        } else if constexpr (IS_F32 && GUARD) {
            const unsigned key = (__float_as_uint((float)e) & ~0x1Fu) | (unsigned)(31 - j);
            if (key > k1) bg = G[j];
            k2 = max(k2, min(k1, key));
            k1 = max(k1, key);
        } else {
            if (e > best) {
                best = e;
                blin = lin0 + (unsigned)(j * RSTEP * F);
                bg = G[j];
            }
        }
    };

#pragma unroll
    for (int j = 0; j < NB; ++j)
        if ((valid >> j) & 1u) track(j, energy(G[j]));

    // fp32: gamma / sum(w) folded into one factor (gamma = 0.5 keeps the
    // products bit-identical); MODE 1 logs p itself
    const T ginv = gamma * inv_tot;
    ArgSlot<T> *asl0 = reinterpret_cast<ArgSlot<T> *>(slots);
    FSE_CLK(4);
    for (int it = 0; it < I; ++it) {
        FSE_CLK(8 + 4 * it);
        // ---- (1) CTA-wide argmax (+ runner-up for the guard), one barrier
        FastSlot<T> *sl = slots + (it & 1) * NWT;
        ArgSlot<T> *asl = asl0 + (it & 1) * NWT;
        // LAZY slots: per-warp maximum keys (double-buffered), then the
        // candidate warps' (lin, g); the key region is 2 NWT x 8 bytes
        KeyT *ska = reinterpret_cast<KeyT *>(reinterpret_cast<unsigned long long *>(slots) + (it & 1) * NWT);
        ArgSlot<T> *skb = reinterpret_cast<ArgSlot<T> *>(reinterpret_cast<unsigned long long *>(slots) + 2 * NWT);
        KeyT wk = 0;
        unsigned *ska32 = reinterpret_cast<unsigned *>(reinterpret_cast<unsigned long long *>(slots) + (it & 1) * NWT);
        unsigned wk32 = 0;
        if constexpr (LAZY64) {
            wk32 = warp_max_u32(hmax);
            if (lane == 0) ska32[warp] = wk32;
        } else if constexpr (LAZY) {
            wk = warp_max_k(energy_key(tmax));
            if (lane == 0) ska[warp] = wk;
        } else if constexpr (IS_F32 && GUARD) {
            const unsigned w1 = warp_max_u32(k1);
            const int wl = __ffs(__ballot_sync(0xffffffffu, k1 == w1)) - 1;
            const unsigned w2 = warp_max_u32(lane == wl ? k2 : k1);
            if (lane == wl) {
                const int jj = 31 - (int)(k1 & 0x1Fu);
                const unsigned lin = (unsigned)((u0 + RSTEP * jj) * F + v);
                sl[warp].key = k1 ? (((unsigned long long)(w1 >> 5) << 32) | (0xFFFFFFFFu - lin)) : 0ull;
                sl[warp].second = w2;
                sl[warp].gre = bg.x;
                sl[warp].gim = bg.y;
            }
        } else {
            const auto key = energy_key(best);
            // one writer: the lane of the warp's first maximum (when the warp
            // has no bin above 0, every lane holds the same empty slot)
#ifndef FSE_ARGMAX_FULL
            if (lane == warp_argmax_lane(key, blin)) {
                ArgSlot<T> mine;
                mine.key = key;
                mine.lin = blin;
#else
            decltype(energy_key(best)) wkey;
            unsigned wlin;
            warp_argmax(key, blin, wkey, wlin);
            if (key == wkey && blin == wlin) {
                ArgSlot<T> mine;
                mine.key = wkey;
                mine.lin = wlin;
#endif
                mine.gre = bg.x;
                mine.gim = bg.y;
                if constexpr (CL > 1) {  // into the slot array of every CTA of the cluster
                    auto cluster = cooperative_groups::this_cluster();
#pragma unroll
                    for (int r = 0; r < CL; ++r) *cluster.map_shared_rank(&asl[gwarp], r) = mine;
                } else {
                    asl[gwarp] = mine;
                }
            }
        }
        if constexpr (CL > 1) cooperative_groups::this_cluster().sync();
        else __syncthreads();
        FSE_CLK(8 + 4 * it + 1);
        int a, b;
        T2 gwin;
        if constexpr (LAZY64) {
            const bool in = lane < NWT;
            const unsigned uk = in ? ska32[lane] : 0u;
            const unsigned H = warp_max_u32(uk);
            if (H == 0) {
                // no energy above 2^-1002 (an all-zero window): the strict '>'
                // scan from -1 keeps (0, 0) (_kernel.pyx:32-44), g = 0
                a = b = 0;
                gwin = T2{0, 0};
            } else {
                if (wk32 == H) {
                    // a candidate warp: its lanes at H resolve their bins with
                    // high word H on the exact keys (first maximum in row-major order)
                    unsigned long long bkey = 0;
                    unsigned mylin = 0xFFFFFFFFu;
                    T2 myg = T2{0, 0};
                    if (hmax == H) {
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
                            const bool inr = (j < NB - 1) || (C::NSEGS % NWT == 0) || (u0 + RSTEP * j < R1);
                            const bool ok = (j == 0 || j == NB - 1) ? ((valid >> j) & 1u) != 0 : inr;
                            const T e = energy(G[j]);
                            const unsigned long long k = energy_key(e);
                            if (ok && (unsigned)(k >> 32) == H && k > bkey) {
                                bkey = k;
                                mylin = lin0 + (unsigned)(j * RSTEP * F);
                                myg = G[j];
                            }
                        }
                    }
                    const unsigned hb = __ballot_sync(0xffffffffu, hmax == H);
                    const int wl = __popc(hb) == 1 ? __ffs(hb) - 1 : warp_argmax_lane(bkey, mylin);
                    if (lane == wl) {
                        ArgSlot<T> mine;
                        mine.key = bkey;
                        mine.lin = mylin;
                        mine.gre = myg.x;
                        mine.gim = myg.y;
                        skb[warp] = mine;
                    }
                }
                __syncthreads();
                const bool cand = in && uk == H;
                const unsigned cb = __ballot_sync(0xffffffffu, cand);
                const int gw = __popc(cb) == 1
                                   ? __ffs(cb) - 1
                                   : warp_argmax_lane(cand ? skb[lane].key : 0ull, cand ? skb[lane].lin : 0xFFFFFFFFu);
                const unsigned glin = skb[gw].lin;
                a = (int)(glin / F);
                b = (int)(glin & (F - 1));
                gwin = T2{skb[gw].gre, skb[gw].gim};
            }
        } else if constexpr (LAZY) {
            const bool in = lane < NWT;
            const KeyT uk = in ? ska[lane] : (KeyT)0;
            const KeyT gk = warp_max_k(uk);
            if (gk == 0) {
                // no bin above 0 (all energies 0 or NaN): the reference's
                // strict-'>' scan from -1 keeps (0, 0) (_kernel.pyx:32-44), g = 0
                a = b = 0;
                gwin = T2{0, 0};
            } else {
                if (wk == gk) {
                    // a candidate warp: its lanes at the maximum find their first
                    // (row-major) bin at that energy; the smallest lin is the warp's
                    unsigned mylin = 0xFFFFFFFFu;
                    T2 myg = T2{0, 0};
                    if (energy_key(tmax) == gk) {
#pragma unroll
                        for (int j = NB - 1; j >= 0; --j) {
                            const bool inr = (j < NB - 1) || (C::NSEGS % NWT == 0) || (u0 + RSTEP * j < R1);
                            const bool ok = (j == 0 || j == NB - 1) ? ((valid >> j) & 1u) != 0 : inr;
                            if (ok && energy_key(energy(G[j])) == gk) {
                                mylin = lin0 + (unsigned)(j * RSTEP * F);
                                myg = G[j];
                            }
                        }
                    }
#ifndef FSE_ARGMAX_FULL
                    // usually one lane of the warp is at the maximum: no REDUX
                    const unsigned hb = __ballot_sync(0xffffffffu, mylin != 0xFFFFFFFFu);
                    const unsigned wl = __popc(hb) == 1 ? __shfl_sync(0xffffffffu, mylin, __ffs(hb) - 1)
                                                        : warp_min_u32(mylin);
#else
                    const unsigned wl = warp_min_u32(mylin);
#endif
                    if (mylin == wl) {
                        ArgSlot<T> mine;
                        mine.key = gk;
                        mine.lin = wl;
                        mine.gre = myg.x;
                        mine.gim = myg.y;
                        skb[warp] = mine;
                    }
                }
                __syncthreads();
                const bool cand = in && uk == gk;
                const unsigned ul = cand ? skb[lane].lin : 0xFFFFFFFFu;
#ifndef FSE_ARGMAX_FULL
                // usually one warp holds the maximum: no REDUX
                const unsigned cb = __ballot_sync(0xffffffffu, cand);
                const unsigned glin = __popc(cb) == 1 ? __shfl_sync(0xffffffffu, ul, __ffs(cb) - 1)
                                                      : warp_min_u32(ul);
#else
                const unsigned glin = warp_min_u32(ul);
#endif
                const int gw = __ffs(__ballot_sync(0xffffffffu, cand && ul == glin)) - 1;
                a = (int)(glin / F);
                b = (int)(glin & (F - 1));
                gwin = T2{skb[gw].gre, skb[gw].gim};
            }
        } else if constexpr (IS_F32 && GUARD) {
            const unsigned long long uk = lane < NW ? sl[lane].key : 0ull;
            const unsigned long long gk = warp_max_key(uk);
            const int gw = __ffs(__ballot_sync(0xffffffffu, uk == gk)) - 1;
            const int lin = (int)(0xFFFFFFFFu - (unsigned)(gk & 0xFFFFFFFFull));
            a = lin / F;
            b = lin - a * F;
            // runner-up energy key: best of the other warps, or the winner warp's second
            const unsigned cand = lane < NW ? (lane == gw ? sl[lane].second : (unsigned)(sl[lane].key >> 32) << 5)
                                            : 0u;
            const unsigned g2 = warp_max_u32(cand);
            const float e1 = __uint_as_float((unsigned)(gk >> 32) << 5);
            const float e2 = __uint_as_float(g2 & ~0x1Fu);
            const float tau = A.tau0 + A.tau1 * (float)it;
            if constexpr (MODE == 0) {
                if (e1 - e2 <= tau * e1) {
                    // near tie: hand the window to the fp64 kernel (uniform exit)
                    if (t == 0) {
                        const int q = atomicAdd(A.redo_count, 1);
                        A.redo_list[q] = entry;
                    }
                    return;
                }
            }
            gwin = *reinterpret_cast<const T2 *>(&sl[gw].gre);
        } else {
            const bool in = lane < NWT;
            const auto uk = in ? asl[lane].key : decltype(asl[0].key)(0);
            const unsigned ul = in ? asl[lane].lin : 0xFFFFFFFFu;
#ifndef FSE_ARGMAX_FULL
            // the winning slot (when no bin is above 0 every slot holds g = 0
            // and lin = none, and the lowest slot wins)
            const int gw = warp_argmax_lane(uk, ul);
            unsigned glin = __shfl_sync(0xffffffffu, ul, gw);
#else
            decltype(asl[0].key) gk;
            unsigned glin;
            warp_argmax(uk, ul, gk, glin);
            // the winning slot (any slot when no bin is above 0: all hold g = 0)
            const int gw = __ffs(__ballot_sync(0xffffffffu, in && ul == glin)) - 1;
#endif
            // no bin above 0 (all energies 0 or NaN): the reference's strict-'>'
            // scan from -1 keeps (0, 0) (_kernel.pyx:32-44), whose g is 0
            if (glin >= (unsigned)(R1 * F)) glin = 0;
            a = (int)(glin / F);
            b = (int)(glin & (F - 1));
            gwin = T2{asl[gw].gre, asl[gw].gim};
        }
        // p = g[a,b] / sum(w) (_kernel.pyx:46-47); fp32 multiplies by 1/sum(w)
        const bool selfc = ((2 * a) & (F - 1)) == 0 && ((2 * b) & (F - 1)) == 0;
        T gpr, gpi;
        if constexpr (IS_F32) {
            gpr = gwin.x * ginv;
            gpi = gwin.y * ginv;
        } else {
#ifndef FSE_P_DIV
            // gamma / sum(w) folded into one factor, as in fp32: p differs from
            // the correctly rounded g / sum(w) of _kernel.pyx:46-47 by an ulp,
            // far below any pick margin; the exact quotient (-DFSE_P_DIV) costs
            // three dependent DFMA on every iteration's critical path
            // (config 4: 551.6 -> 542.8 ms without it)
            gpr = gwin.x * ginv;
            gpi = gwin.y * ginv;
#else
            gpr = gamma * div_by(gwin.x, tot, inv_tot);
            gpi = gamma * div_by(gwin.y, tot, inv_tot);
#endif
        }
        if constexpr (MODE == 1) {
            if (gwarp == 0 && lane == 0) {
                picks_out[2 * it] = a;
                picks_out[2 * it + 1] = b;
                if constexpr (IS_F32) {
                    plog[2 * it] = gwin.x * inv_tot;
                    plog[2 * it + 1] = gwin.y * inv_tot;
                } else {
                    plog[2 * it] = div_by(gwin.x, tot, inv_tot);
                    plog[2 * it + 1] = div_by(gwin.y, tot, inv_tot);
                }
            }
        }
        FSE_CLK(8 + 4 * it + 2);
        // self-conjugate: gamma * Re(p) * W[k - j] == (gamma Re(p) / 2) (W[k-j] + W[k+j])
        if (selfc) {
            gpr = gpr * (T)0.5;
            gpi = (T)0;
        }

        // ---- (2) log the pick for the block model (synthesised after the loop)
        if constexpr (MODE == 0) {
            if (gwarp == 0 && lane == 0) hist[it] = PickRec<T>{a, b, gpr, gpi};
        }
        if (it + 1 == I) break;  // the last spectrum update is never observed

        // ---- (3) spectrum update by the shifted weight spectrum + next argmax
        const int cm = (v - b) & (F - 1), cp = (v + b) & (F - 1);
        // EXT: rows u-a and u+a are in the extended plane as they are.
        // plain: row (u0 - a + RSTEP j) mod F wraps for the first jl bins (below
        // 0); row u0 + a + RSTEP j <= F is stored as it is (row F = row 0).
        const int x0 = u0 - a, y0 = u0 + a;
        const T2 *lo = Wext + (C::EXT ? (x0 + F / 2) * F : x0 * F) + cm;
        const T2 *hi = Wext + (C::EXT ? (y0 + F / 2) * F : y0 * F) + cp;
        const T2 *loW = lo + F * F;  // plain plane: wrapped base
        const int jl = x0 < 0 ? (RSTEP - 1 - x0) / RSTEP : 0;
        // HALF: row x0 + RSTEP j < 0 reads conj W[-x0 - RSTEP j][(b - v) mod F]
        // (j < jl), row y0 + RSTEP j > F/2 reads conj W[F - y0 - RSTEP j][(-v - b) mod F]
        // (j >= jh); offsets, not pointers, since the bases may lie outside the plane
        const int offLD = x0 * F + cm, offLR = -x0 * F + ((b - v) & (F - 1));
        const int offHD = y0 * F + cp, offHR = (F - y0) * F + ((-v - b) & (F - 1));
        const int jh = F / 2 - y0 >= 0 ? (F / 2 - y0) / RSTEP + 1 : 0;
        k1 = 0;
        k2 = 0;
        best = (T)0;
        blin = 0xFFFFFFFFu;
        tmax = (T)0;
        hmax = 0;
        const T2 mS = T2{-gpr, -gpr}, qv = T2{gpi, -gpi};
        // loads of a group of LG bins are issued before its math (smem latency);
        // measured on config 4: fp32 LG 1/2/3/4/6/11 = 284.2/283.4/289.2/287.5/
        // 292.5/302.4 ms, fp64 LG 1/2/3 = 554.4/558.8/554.9 ms
#ifndef FSE_LG32
#define FSE_LG32 2
#endif
#ifndef FSE_LG64
#define FSE_LG64 1
#endif
        constexpr int LG = C::LGC > 0 ? C::LGC : (IS_F32 ? FSE_LG32 : FSE_LG64);
#pragma unroll
        for (int j0 = 0; j0 < NB; j0 += LG) {
            T2 wl[LG], wh[LG];
#pragma unroll
            for (int q = 0; q < LG; ++q) {
                const int j = j0 + q;
                const bool inr = j < NB && ((j < NB - 1) || (C::NSEGS % NWT == 0) || (u0 + RSTEP * j < R1));
                if (inr) {
                    if constexpr (C::HALF) {
                        const bool rl = j < jl, rh = j >= jh;
                        wl[q] = Wext[rl ? offLR - j * RSTEP * F : offLD + j * RSTEP * F];
                        wh[q] = Wext[rh ? offHR - j * RSTEP * F : offHD + j * RSTEP * F];
                        if (rl) wl[q].y = -wl[q].y;
                        if (rh) wh[q].y = -wh[q].y;
                    } else if constexpr (C::EXT) {
                        wl[q] = lo[j * RSTEP * F];
                        wh[q] = hi[j * RSTEP * F];
                    } else {
                        // plain plane, narrow-level variant: row (x0 + RSTEP j) mod F by
                        // masking the byte offset (an add and an AND per bin instead of the
                        // compare and two-base select).  Only there: config 2 7.81 -> 7.73 ms,
                        // but the 6-warp throughput kernel loses 8% with it (559 vs 519 ms on
                        // config 4: the two dependent ALU operations sit in front of every
                        // u-a gather), profiles/r4/ab_loop/
                        if constexpr (C::LGC > 0 && !IS_F32) {
                            static_assert(((F * F * sizeof(T2)) & (F * F * sizeof(T2) - 1)) == 0, "power-of-two plane");
                            const unsigned ob = (unsigned)((x0 * F + cm) * (int)sizeof(T2));
                            wl[q] = *reinterpret_cast<const T2 *>(reinterpret_cast<const char *>(Wext) +
                                                                  ((ob + (unsigned)(j * RSTEP * F * sizeof(T2))) &
                                                                   (unsigned)(F * F * sizeof(T2) - 1)));
                        } else {
                            wl[q] = (j < jl ? loW : lo)[j * RSTEP * F];
                        }
                        wh[q] = hi[j * RSTEP * F];
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < LG; ++q) {
                const int j = j0 + q;
                const bool inr = j < NB && ((j < NB - 1) || (C::NSEGS % NWT == 0) || (u0 + RSTEP * j < R1));
                if (inr) {
                    if constexpr (IS_F32) G[j] = spectral_update_bc(G[j], wl[q], wh[q], -gpr, gpi);
                    else G[j] = spectral_update(G[j], wl[q], wh[q], mS, qv);
                    const T e = energy(G[j]);
                    if (j == 0 || j == NB - 1) {
                        if ((valid >> j) & 1u) track(j, e);
                    } else {
                        track(j, e);
                    }
                }
            }
        }
    }

    FSE_CLK(5);
    // ---- model over the block: sum_it 2 Re(gamma p_it e^{+j 2 pi (a i + b j)/F}),
    // fse.py:159 restricted to the block rect
    if constexpr (MODE == 0) {
        __syncthreads();
        if (picks_out && crank == 0)
            for (int i = t; i < I; i += NT) {
                picks_out[2 * i] = hist[i].a;
                picks_out[2 * i + 1] = hist[i].b;
            }
        // every thread sums the iterations it = r (mod nsub) of one sample q
        // (nsub = NT / samples subsets), then one thread per sample adds the
        // nsub partials in subset order; the W plane is dead, so the partials
        // reuse its bytes.  More samples than threads: all iterations per sample.
        const int nsamp = bh * bw;
        IT *img = reinterpret_cast<IT *>(fd->image);
        auto model = [&](int q, int r0, int step) -> T {
            const int mi = br0 + q / bw, mj = bc0 + q % bw;
            T acc = (T)0;
            for (int it = r0; it < I; it += step) {
                const PickRec<T> h = hist[it];
                const T2 ph = tw[(h.a * mi + h.b * mj) & (F - 1)];
                acc += (T)2 * (h.gpr * ph.x - h.gpi * ph.y);
            }
            return acc;
        };
        // write-back of the block's LOST samples (conceal.py:61-66)
        const int brow = blk / A.cols;
        IT *pu = (A.peer_up && brow < A.peer_up_end) ? reinterpret_cast<IT *>(A.peer_up) : nullptr;
        IT *pd = (A.peer_down && brow >= A.peer_down_begin) ? reinterpret_cast<IT *>(A.peer_down) : nullptr;
        auto store = [&](int q, T val) {
            const size_t off = (size_t)(wr0 + br0 + q / bw) * A.W + (wc0 + bc0 + q % bw);
            if (fd->mask[off] == FSE_LOST) {
                img[off] = (IT)val;
                // halo rows straight into the neighbour's frame over NVLink
                if (pu) pu[off] = (IT)val;
                if (pd) pd[off] = (IT)val;
            }
        };
        if (crank == 0) {  // the cluster's CTA 0 writes the block
            // the subset count depends on F and the block only (not on the
            // warps of this variant), so every variant of one F sums the model
            // in the same order and gives bit-identical samples
            if (nsamp <= C::NSUB_BASE) {
                const int nsub = C::NSUB_BASE / nsamp, q = t % nsamp, r = t / nsamp;
                T *red2 = reinterpret_cast<T *>(big);
                if (r < nsub) red2[r * nsamp + q] = model(q, r, nsub);
                __syncthreads();
                if (t < nsamp) {
                    T v = (T)0;
                    for (int k = 0; k < nsub; ++k) v += red2[k * nsamp + t];
                    store(t, v);
                }
            } else {
                for (int q = t; q < nsamp; q += NT) store(q, model(q, 0, 1));
            }
            // peer stores visible system-wide before this kernel completes (the
            // stream's next op signals the neighbour)
            if (pu || pd) __threadfence_system();
        }
    }
    FSE_CLK(6);
    // keep this CTA's shared memory alive until the cluster is done with it
    if constexpr (CL > 1) cooperative_groups::this_cluster().sync();
}

// (The two code paths as separate __noinline__ functions were tried: the
// by-reference kernel parameters then live in local memory and the computing
// path spills 220 B instead of 64 B.)
// TWIN: the kernel also holds the cached-W code path (launched for sessions
// with a weight-spectrum cache).  Sessions without one launch the TWIN = false
// instance, which is the kernel as it was before the cache existed: with the
// twin inlined beside it ptxas schedules the computing path differently (its
// x row pass 12.9 k -> 36.8 k cycles per window, +3% on config 4).
template <class C, int MODE, bool GUARD, bool TWIN = false>
__global__ void __launch_bounds__(C::NT, C::MINB) fse_fast_kernel(const FastArgs A, const FastLayout L) {
    extern __shared__ __align__(128) unsigned char sm[];
    // programmatic dependent launch (level launches, fse_inst_fast.cu): let the
    // next level's grid be scheduled now, and wait for the previous level's
    // grid (complete, memory visible) before touching global memory -- the
    // launch gap between dependent levels overlaps this level's work
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr (TWIN) {
        static_assert(MODE == 0 && !GUARD && C::CL == 1, "cached W: plain pipeline levels");
        // a window whose W is in the session's cache takes the twin code path
        // without the weight half of the set-up (uniform over the CTA)
        const int wc = A.wslot ? A.wslot[blockIdx.x] : -1;
        if (wc >= 0) {
            fast_window<C, MODE, GUARD, typename C::T, true>(A, L, blockIdx.x, sm, make_int2(-1, -1), wc);
            return;
        }
    }
    fast_window<C, MODE, GUARD, typename C::T>(A, L, blockIdx.x, sm);
}

// Cluster variant: CL CTAs (one window) per cluster, window = blockIdx.x / CL.
template <class C>
__global__ void __cluster_dims__(C::CL, 1, 1) __launch_bounds__(C::NT)
    fse_fast_cluster_kernel(const FastArgs A, const FastLayout L) {
    extern __shared__ __align__(128) unsigned char sm[];
    fast_window<C, 0, false, typename C::T>(A, L, blockIdx.x / C::CL, sm);
}

// Persistent variant over a device-side list (the fp64 redo of guarded windows
// of an fp32 image: IT = float, compute type C::T = double).
template <class C, typename IT>
__global__ void __launch_bounds__(C::NT) fse_fast_redo_kernel(const FastArgs A, const FastLayout L) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int n = *A.count;
    for (int e = blockIdx.x; e < n; e += gridDim.x) {
        fast_window<C, 0, false, IT>(A, L, e, sm);
        __syncthreads();
    }
}

// Persistent dataflow execution.  The level barrier is
// replaced by per-block dependency counters over the rank-overlap DAG: block o
// depends on every processed block of lower rank within the dependency radius
// (its window reads their samples).  dataflow_init_kernel counts those
// dependencies and enqueues the blocks that have none; the persistent kernel
// pops ready blocks from a global queue, fits them, and on completion
// decrements its dependents' counters, enqueueing each one whose count reaches
// zero.  A CTA never holds a block that is not ready, so resident CTAs only wait
// for the queue to grow, which the running CTAs guarantee: no deadlock.
// Ordering: write-back -> bar.sync -> acq_rel counter decrement (release
// sequence) -> st.release of the queue slot -> consumer ld.acquire.
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// One thread per entry: dependency count; blocks without dependencies are queued.
static __global__ void dataflow_init_kernel(const FastArgs A) {
    const int nb = A.rows * A.cols;
    const int R = A.R;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.total; e += gridDim.x * blockDim.x) {
        const int2 en = A.entries[e];
        const int *rank = A.frames[en.x].rank;
        const int r = en.y / A.cols, c = en.y - r * A.cols;
        const int myrank = rank[en.y];
        int deps = 0;
        for (int rr = max(0, r - R); rr <= min(A.rows - 1, r + R); ++rr)
            for (int cc = max(0, c - R); cc <= min(A.cols - 1, c + R); ++cc)
                deps += rank[rr * A.cols + cc] < myrank;
        A.done[(size_t)en.x * nb + en.y] = deps;
        if (deps == 0) {
            const int k = atomicAdd(A.next + 1, 1);  // queue tail
            A.queue[k] = en.x * nb + en.y;          // consumers start after this kernel
        }
    }
}

template <class C, typename IT>
__global__ void __launch_bounds__(C::NT) fse_fast_dataflow_kernel(const FastArgs A, const FastLayout L) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ int s_code;
    const int t = threadIdx.x;
    const int nb = A.rows * A.cols;
    const int R = A.R, side = 2 * R + 1;
    for (;;) {
        if (t == 0) {
            const int i = atomicAdd(A.next, 1);  // queue head
            int code = -2;
            if (i < A.total) {
                while ((code = ld_acquire(A.queue + i)) < 0) __nanosleep(100);
            }
            s_code = code;
        }
        __syncthreads();
        const int code = s_code;
        if (code == -2) break;
        const int2 en = make_int2(code / nb, code - (code / nb) * nb);
        fast_window<C, 0, false, IT>(A, L, 0, sm, en);
        __syncthreads();  // the CTA's write-back stores precede the releases below
        const int *rank = A.frames[en.x].rank;
        const int r = en.y / A.cols, c = en.y - r * A.cols;
        const int myrank = rank[en.y];
        int *cnt = A.done + (size_t)en.x * nb;
        for (int q = t; q < side * side; q += C::NT) {
            const int rr = r - R + q / side, cc = c - R + q % side;
            if (rr < 0 || rr >= A.rows || cc < 0 || cc >= A.cols) continue;
            const int o = rr * A.cols + cc;
            const int ro = rank[o];
            if (o == en.y || ro <= myrank || ro == 0x7FFFFFFF) continue;
            if (atom_add_acq_rel(cnt + o, -1) == 1) {
                const int k = atomicAdd(A.next + 1, 1);
                st_release(A.queue + k, en.x * nb + o);
            }
        }
    }
}

// Host launchers (fse_inst_fast.cu).  dtype FSE_F32/FSE_F64, F = 32/64 (and 128 in fp32).
int fast_supported(int dtype, int F, int Mmax, int Nmax, int model_n, int iterations);
int fast_level(int dtype, int F, bool guard, const FastArgs &a, int grid, int Mmax, int Nmax,
               int model_n, cudaStream_t s);
int fast_dataflow(int dtype, int F, const FastArgs &a, int Mmax, int Nmax, int model_n,
                  cudaStream_t s);
int fast_redo(int F, const FastArgs &a, int max_entries, int Mmax, int Nmax, int model_n,
              cudaStream_t s);
int fast_windows(int dtype, int F, const FastArgs &a, int grid, cudaStream_t s);
// W-cache producer (MODE 2): plane p < *a.count from window a.entries[a.wrep[p]], grid = plane capacity
int fast_wplanes(int dtype, int F, const FastArgs &a, int grid, int Mmax, int Nmax, int model_n,
                 cudaStream_t s);

}  // namespace fse
