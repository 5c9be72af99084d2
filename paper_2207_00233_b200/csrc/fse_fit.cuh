// Per-window FSE model fit on sm_100a: one CTA owns one extrapolation window.
//
// Reference algorithm: fsefill._kernel.run_fse / _iterate
// (/root/reference/pkg/src/fsefill/_kernel.pyx:14-187).  Per window:
//   x = w * select(w > 0, v, 0);  g = DFT_F(x);  W = DFT_F(w)     (_kernel.pyx:144-148)
//   repeat I times:
//     (a,b) = argmax |g|^2, first maximum in row-major order     (:32-44)
//     p = g[a,b] / sum(w)                                          (:46-47)
//     self-conjugate (a,b):  g -= gamma*Re(p)*W[k-(a,b)]           (:50-64)
//     else                   g -= gamma*(p W[k-(a,b)] + conj(p) W[k+(a,b)])  (:65-97)
//
// B200 layout:
//   * g lives in REGISTERS, only the non-redundant half spectrum (rows
//     0..F1/2 of the F1 x F2 plane: w*r is real, so g[-k] = conj g[k] and the
//     update preserves that).  17*F1*(F2/2+1) counted FLOPs per iteration.
//   * W (the window's weight spectrum) lives in SHARED memory as a full plane
//     (or, when that does not fit, the half plane plus conjugate reflection);
//     every bin gathers two shifted W entries per iteration — the shared-memory
//     crossbar (128 B/clk/SM) is the practical roofline of this kernel.
//   * Fast path (F = 32/64/128): warp w owns row segment (w % SEG) of rows
//     w/SEG + (NW/SEG)*j, so lane-consecutive bins hit consecutive W addresses
//     (conflict-free) and row indices are warp-uniform.
//   * argmax: per-thread running max, warp REDUX on a packed (|g|^2, index)
//     key, one __syncthreads per iteration with double-buffered slots; ties go
//     to the smallest row-major index as in the reference.
//   * DFT set-up: direct separable DFT against sincospi twiddle tables
//     (column pass over the M non-zero rows, then row pass over the owned
//     bins); the weight spectrum is mirrored into the full plane by symmetry.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fse {

template <typename T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };

// Pack (energy, row-major bin index) into an order-preserving 64-bit key:
// larger energy wins, ties go to the smaller index.
__device__ __forceinline__ unsigned long long pack_key(double e, int lin) {
    unsigned long long bits = (unsigned long long)__double_as_longlong(e);
    return (bits & ~0xFFFFull) | (unsigned long long)(0xFFFF - lin);
}
__device__ __forceinline__ unsigned long long pack_key(float e, int lin) {
    return ((unsigned long long)__float_as_uint(e) << 32) | (unsigned long long)(0xFFFF - lin);
}

__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
    unsigned hi = (unsigned)(k >> 32);
    unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    unsigned lo = hi == mhi ? (unsigned)k : 0u;
    unsigned mlo = __reduce_max_sync(0xffffffffu, lo);
    return ((unsigned long long)mhi << 32) | mlo;
}

template <typename T> struct Slot {
    unsigned long long key;
    T pre, pim;
};

// Shared-memory carve-up, identical on host and device.
struct SmemLayout {
    size_t tw1, tw2, slots, red, model, big, off_Yx, off_Yw, big_bytes, dbg_res, dbg_w, total;
};

template <typename T>
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename T, typename ST>
__host__ __device__ inline SmemLayout smem_layout(int Mmax, int Nmax, int F1max, int F2max,
                                                  int NW, int model_n, bool debug, bool fullw) {
    SmemLayout L;
    size_t o = 0;
    const size_t cT = 2 * sizeof(T), cS = 2 * sizeof(ST);
    L.tw1 = o; o = align16<T>(o + (size_t)F1max * 2 * sizeof(T));
    L.tw2 = o; o = align16<T>(o + (size_t)F2max * 2 * sizeof(T));
    L.slots = o; o = align16<T>(o + 2 * (size_t)NW * sizeof(Slot<T>));
    L.red = o; o = align16<T>(o + (size_t)(NW + 2) * sizeof(double));
    L.model = o; o = align16<T>(o + (size_t)(model_n > 0 ? model_n : 1) * sizeof(T));
    o = (o + 127) & ~size_t(127);
    L.big = o;
    const size_t R1 = (size_t)F1max / 2 + 1;
    const size_t xs_ws = align16<T>(2 * (size_t)Mmax * Nmax * sizeof(ST));
    const size_t ybytes = align16<T>(R1 * (size_t)Nmax * cS);
    const size_t whalf = align16<T>(R1 * (size_t)F2max * cT);
    const size_t wplane = fullw ? (size_t)F1max * F2max * cT : whalf;
    L.off_Yx = xs_ws;
    L.off_Yw = L.off_Yx + ybytes > whalf ? L.off_Yx + ybytes : whalf;
    L.big_bytes = L.off_Yw + ybytes > wplane ? L.off_Yw + ybytes : wplane;
    o = align16<T>(L.big + L.big_bytes);
    L.dbg_res = o;
    if (debug) o = align16<T>(o + (size_t)F1max * F2max * sizeof(T));
    L.dbg_w = o;
    if (debug) o = align16<T>(o + (size_t)Mmax * Nmax * sizeof(T));
    L.total = o;
    return L;
}

// Compile-time description of a kernel variant.
//   F  = 32/64/128: square power-of-two DFT with the warp-row bin layout;
//   F  = 0: runtime F1 x F2 (any size, e.g. the reference's DFT = window shape).
template <typename T_, typename ST_, int F_, int NW_, bool FULLW_>
struct Cfg {
    using T = T_;
    using ST = ST_;
    static constexpr int F = F_;
    static constexpr int NW = NW_;
    static constexpr int NT = NW_ * 32;
    static constexpr bool FULLW = FULLW_;
    static constexpr int SEG = F_ > 0 ? F_ / 32 : 1;
    static constexpr int RPR = F_ > 0 ? NW_ / SEG : 1;  // rows per round
    static constexpr int NB = F_ > 0 ? (F_ / 2 + 1 + RPR - 1) / RPR : 16;
    static_assert(F_ == 0 || (F_ >= 32 && (F_ & (F_ - 1)) == 0), "F must be 0 or a power of two >= 32");
    static_assert(F_ == 0 || NW_ % (F_ > 0 ? F_ / 32 : 1) == 0, "NW must be a multiple of F/32");
};

}  // namespace fse
