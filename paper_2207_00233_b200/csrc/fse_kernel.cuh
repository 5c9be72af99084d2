// Kernel template + launcher shared by the per-variant translation units
// (fse_inst_*.cu instantiate launch_variant<> for one dtype each, so nvcc
// compiles the variants in parallel).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <string>
#include <type_traits>

#include "fse_common.h"
#include "fse_fit.cuh"

namespace fse {

extern std::atomic<long long> g_launches;

struct FrameDesc {
    void *image;
    const uint8_t *mask;
    uint8_t *mask_out;
    const int32_t *rank;
};

// Arguments of one launch.  MODE 0 = pipeline level, MODE 1 = window operator.
struct KArgs {
    // pipeline
    const FrameDesc *frames;
    const int2 *entries;
    int H, W, B, d, rows, cols;
    double delta;
    const double *decay;
    int decay_dim;
    // window operator
    const void *values, *weights;
    void *plog, *energies, *residual;
    // both
    int M, N;      // window operator: window shape; pipeline: unused
    int F1, F2;    // DFT size (0 = window shape, pipeline + generic only)
    int iterations;
    double gamma;
    int32_t *picks;
};

#define FSE_CUDA_TRY(expr)                                                          \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess)                                                      \
            return fail(FSE_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// ---------------------------------------------------------------------------
// The kernel.

template <class C, int MODE, bool DEBUG>
__global__ void __launch_bounds__(C::NT) fse_window_kernel(const KArgs A, const SmemLayout L) {
    using T = typename C::T;
    using ST = typename C::ST;
    using T2 = typename V2<T>::type;
    using S2 = typename V2<ST>::type;
    constexpr int NT = C::NT, NW = C::NW, NB = C::NB, CF = C::F;
    extern __shared__ __align__(128) unsigned char sm[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    // ---- window geometry (grid.py:108-135: block +- d, clipped to the image)
    int M, N, F1, F2, br0 = 0, bc0 = 0, bh = 0, bw = 0, wr0 = 0, wc0 = 0, frame = 0, blk = 0;
    const FrameDesc *fd = nullptr;
    if constexpr (MODE == 0) {
        const int2 e = A.entries[blockIdx.x];
        frame = e.x;
        blk = e.y;
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
        F1 = A.F1 ? A.F1 : M;
        F2 = A.F2 ? A.F2 : N;
    } else {
        M = A.M;
        N = A.N;
        F1 = A.F1;
        F2 = A.F2;
    }
    if constexpr (CF > 0) {
        F1 = CF;
        F2 = CF;
    }
    const int R1 = F1 / 2 + 1;

    S2 *tw1 = reinterpret_cast<S2 *>(sm + L.tw1);
    S2 *tw2 = (CF > 0) ? tw1 : reinterpret_cast<S2 *>(sm + L.tw2);
    Slot<T> *slots = reinterpret_cast<Slot<T> *>(sm + L.slots);
    double *red = reinterpret_cast<double *>(sm + L.red);
    T *model = reinterpret_cast<T *>(sm + L.model);
    unsigned char *big = sm + L.big;
    ST *xs = reinterpret_cast<ST *>(big);
    ST *ws = xs + M * N;
    S2 *Yx = reinterpret_cast<S2 *>(big + L.off_Yx);
    S2 *Yw = reinterpret_cast<S2 *>(big + L.off_Yw);
    T2 *Wp = reinterpret_cast<T2 *>(big);
    T *dres = reinterpret_cast<T *>(sm + L.dbg_res);
    T *dw = reinterpret_cast<T *>(sm + L.dbg_w);

    // ---- unit-circle tables e^{+j 2 pi k / F} (forward DFT uses the conjugate)
    for (int k = t; k < F1; k += NT) {
        double s, c;
        sincospi(2.0 * k / F1, &s, &c);
        tw1[k] = S2{(ST)c, (ST)s};
    }
    if (CF == 0)
        for (int k = t; k < F2; k += NT) {
            double s, c;
            sincospi(2.0 * k / F2, &s, &c);
            tw2[k] = S2{(ST)c, (ST)s};
        }

    // ---- staging: classes -> weights (fse.py:105-119), x = w * select(w>0, v, 0)
    double wsum = 0.0, e0 = 0.0;
    if constexpr (MODE == 0) {
        const int myrank = fd->rank[blk];
        const T *img = reinterpret_cast<const T *>(fd->image);
        for (int idx = t; idx < M * N; idx += NT) {
            const int i = idx / N, j = idx - i * N;
            const int y = wr0 + i, x = wc0 + j;
            const uint8_t s = fd->mask[(size_t)y * A.W + x];
            const double dec = A.decay[abs(2 * i - (M - 1)) * A.decay_dim + abs(2 * j - (N - 1))];
            double w;
            if (s == FSE_LOST) {
                const int owner = (y / A.B) * A.cols + x / A.B;
                // R iff the owner block was written by an earlier batch (snapshot
                // semantics, conceal.py:148-163); BI / BO otherwise (weight 0)
                w = (owner != blk && fd->rank[owner] < myrank) ? A.delta * dec : 0.0;
            } else if (s == FSE_RECONSTRUCTED) {
                w = A.delta * dec;
            } else {
                w = dec;
            }
            const double v = (double)img[(size_t)y * A.W + x];
            xs[idx] = w > 0.0 ? (ST)(w * v) : (ST)0;
            ws[idx] = (ST)w;
            wsum += w;
        }
        for (int q = t; q < bh * bw; q += NT) model[q] = (T)0;
    } else {
        const T *val = reinterpret_cast<const T *>(A.values) + (size_t)blockIdx.x * M * N;
        const T *wgt = reinterpret_cast<const T *>(A.weights) + (size_t)blockIdx.x * M * N;
        for (int idx = t; idx < M * N; idx += NT) {
            const double w = (double)wgt[idx];
            const double r0 = w > 0.0 ? (double)val[idx] : 0.0;
            xs[idx] = (ST)(w * r0);
            ws[idx] = (ST)w;
            wsum += w;
            if constexpr (DEBUG) {
                e0 += w * r0 * r0;
                dw[idx] = (T)w;
            }
        }
        if constexpr (DEBUG) {
            for (int idx = t; idx < F1 * F2; idx += NT) {
                const int i = idx / F2, j = idx - i * F2;
                T r0 = (T)0;
                if (i < M && j < N) {
                    const T w = wgt[i * N + j];
                    r0 = w > (T)0 ? val[i * N + j] : (T)0;
                }
                dres[idx] = r0;
            }
        }
    }
    // block sums of sum(w) (and the initial energy in debug mode)
    for (int off = 16; off; off >>= 1) {
        wsum += __shfl_xor_sync(0xffffffffu, wsum, off);
        if (DEBUG) e0 += __shfl_xor_sync(0xffffffffu, e0, off);
    }
    if (lane == 0) red[warp] = wsum;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += red[w];
        red[NW] = s;
    }
    __syncthreads();
    const double total = red[NW];
    if constexpr (DEBUG) {
        if (lane == 0) red[warp] = e0;
        __syncthreads();
        if (t == 0) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += red[w];
            reinterpret_cast<T *>(A.energies)[(size_t)blockIdx.x * (A.iterations + 1)] = (T)s;
        }
        __syncthreads();
    }

    // ---- DFT pass 1 (columns): Y[k1][n] = sum_m x[m][n] e^{-j2pi k1 m / F1}, k1 <= F1/2
    for (int o = t; o < R1 * N; o += NT) {
        const int k1 = o / N, n = o - k1 * N;
        ST xr = 0, xi = 0, wr = 0, wi = 0;
        int k = 0;
        for (int m = 0; m < M; ++m) {
            const S2 tw = tw1[k];
            const ST xv = xs[m * N + n], wv = ws[m * N + n];
            xr = fma(xv, tw.x, xr);
            xi = fma(-xv, tw.y, xi);
            wr = fma(wv, tw.x, wr);
            wi = fma(-wv, tw.y, wi);
            k += k1;
            if (k >= F1) k -= F1;
        }
        Yx[o] = S2{xr, xi};
        Yw[o] = S2{wr, wi};
    }
    __syncthreads();

    // ---- bin ownership
    // fast layout: warp-row segments; generic: linear bins i = t + NT*j
    const int seg = warp % C::SEG;
    const int u0 = warp / C::SEG;
    const int vfix = seg * 32 + lane;
    int gu[CF > 0 ? 1 : NB], gv[CF > 0 ? 1 : NB];
    if constexpr (CF == 0) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int i = t + NT * j;
            gu[j] = i / F2;
            gv[j] = i - gu[j] * F2;
        }
    }
    auto bin_u = [&](int j) -> int { if constexpr (CF > 0) return u0 + C::RPR * j; else return gu[j]; };
    auto bin_v = [&](int j) -> int { if constexpr (CF > 0) return vfix; else return gv[j]; };
    auto bin_ok = [&](int j) -> bool {
        if constexpr (CF > 0) return u0 + C::RPR * j < R1;
        else return gu[j] < R1;
    };

    // ---- DFT pass 2 (rows) for the owned bins: g into registers
    T g_re[NB], g_im[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        g_re[j] = (T)0;
        g_im[j] = (T)0;
        if (bin_ok(j)) {
            const int u = bin_u(j), v = bin_v(j);
            ST ar = 0, ai = 0;
            int k = 0;
            const S2 *yrow = Yx + u * N;
            for (int n = 0; n < N; ++n) {
                const S2 y = yrow[n], tw = tw2[k];
                ar = fma(y.x, tw.x, fma(y.y, tw.y, ar));
                ai = fma(y.y, tw.x, fma(-y.x, tw.y, ai));
                k += v;
                if (k >= F2) k -= F2;
            }
            g_re[j] = (T)ar;
            g_im[j] = (T)ai;
        }
    }
    __syncthreads();  // xs, ws, Yx dead: the W half plane may overwrite them
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        if (bin_ok(j)) {
            const int u = bin_u(j), v = bin_v(j);
            ST ar = 0, ai = 0;
            int k = 0;
            const S2 *yrow = Yw + u * N;
            for (int n = 0; n < N; ++n) {
                const S2 y = yrow[n], tw = tw2[k];
                ar = fma(y.x, tw.x, fma(y.y, tw.y, ar));
                ai = fma(y.y, tw.x, fma(-y.x, tw.y, ai));
                k += v;
                if (k >= F2) k -= F2;
            }
            Wp[u * F2 + v] = T2{(T)ar, (T)ai};
        }
    }
    __syncthreads();
    if constexpr (C::FULLW) {  // W[-k] = conj W[k] fills rows R1..F1-1
        for (int idx = t; idx < (F1 - R1) * F2; idx += NT) {
            const int r = R1 + idx / F2, c = idx % F2;
            const T2 s = Wp[(F1 - r) * F2 + (c == 0 ? 0 : F2 - c)];
            Wp[r * F2 + c] = T2{s.x, -s.y};
        }
        __syncthreads();
    }

    // W lookup at (r, c) taken modulo the plane
    auto Wat = [&](int r, int c) -> T2 {
        if constexpr (C::FULLW) {
            return Wp[r * F2 + c];
        } else {
            if (r < R1) return Wp[r * F2 + c];
            const T2 s = Wp[(F1 - r) * F2 + (c == 0 ? 0 : F2 - c)];
            return T2{s.x, -s.y};
        }
    };

    // ---- running argmax over the owned bins
    auto local_key = [&]() -> unsigned long long {
        T best = (T)-1;
        int bj = -1;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            if (bin_ok(j)) {
                const T e = g_re[j] * g_re[j] + g_im[j] * g_im[j];
                if (e > best) {
                    best = e;
                    bj = j;
                }
            }
        }
        if (bj < 0) return 0ull;
        int lin = 0;
#pragma unroll
        for (int j = 0; j < NB; ++j)
            if (j == bj) lin = bin_u(j) * F2 + bin_v(j);
        return pack_key(best, lin);
    };
    unsigned long long key = local_key();

    const T gamma = (T)A.gamma;
    const T tot = (T)total;
    const int I = A.iterations;
    int32_t *picks_out = nullptr;
    T *plog = nullptr;
    if constexpr (MODE == 0) {
        if (A.picks) picks_out = A.picks + ((size_t)frame * A.rows * A.cols + blk) * (size_t)I * 2;
    } else {
        picks_out = A.picks + (size_t)blockIdx.x * I * 2;
        plog = reinterpret_cast<T *>(A.plog) + (size_t)blockIdx.x * I * 2;
    }

    for (int it = 0; it < I; ++it) {
        // ---- (1) global argmax: warp REDUX, one barrier, every warp re-reduces the slots
        Slot<T> *sl = slots + (it & 1) * NW;
        const unsigned long long wk = warp_max_key(key);
        const unsigned writers = __ballot_sync(0xffffffffu, key == wk);
        if (lane == __ffs(writers) - 1) {
            // projection coefficient of this warp's best bin (_kernel.pyx:46-47)
            const int lin = 0xFFFF - (int)(wk & 0xFFFFull);
            T pr = (T)0, pi = (T)0;
#pragma unroll
            for (int j = 0; j < NB; ++j)
                if (bin_ok(j) && bin_u(j) * F2 + bin_v(j) == lin) {
                    pr = g_re[j];
                    pi = g_im[j];
                }
            sl[warp].key = wk;
            sl[warp].pre = pr / tot;
            sl[warp].pim = pi / tot;
        }
        __syncthreads();
        const unsigned long long uk = lane < NW ? sl[lane].key : 0ull;
        const unsigned long long gk = warp_max_key(uk);
        const int wl = __ffs(__ballot_sync(0xffffffffu, uk == gk)) - 1;
        const T pre = sl[wl].pre, pim = sl[wl].pim;
        const int lin = 0xFFFF - (int)(gk & 0xFFFFull);
        const int a = lin / F2, b = lin - a * F2;
        const bool selfc = ((2 * a) % F1 == 0) && ((2 * b) % F2 == 0);
        const T gpr = gamma * pre, gpi = gamma * pim;
        if (t == 0 && picks_out) {
            picks_out[2 * it] = a;
            picks_out[2 * it + 1] = b;
            if (plog) {
                plog[2 * it] = pre;
                plog[2 * it + 1] = pim;
            }
        }

        // ---- (2) model over the block (MODE 0) / residual + energy (DEBUG)
        auto phase = [&](int i, int j) -> S2 {  // e^{+j2pi(a i/F1 + b j/F2)}
            if constexpr (CF > 0) {
                return tw1[(a * i + b * j) & (CF - 1)];
            } else {
                const S2 p = tw1[(a * i) % F1], q = tw2[(b * j) % F2];
                return S2{p.x * q.x - p.y * q.y, p.x * q.y + p.y * q.x};
            }
        };
        if constexpr (MODE == 0) {
            for (int q = t; q < bh * bw; q += NT) {
                const int i = br0 + q / bw, j = bc0 + q % bw;
                const S2 ph = phase(i, j);
                const T c = (T)ph.x, s = (T)ph.y;
                model[q] += selfc ? gpr * c : (T)2 * (gpr * c - gpi * s);
            }
        }
        if constexpr (DEBUG) {
            double el = 0.0;
            for (int idx = t; idx < F1 * F2; idx += NT) {
                const int i = idx / F2, j = idx - i * F2;
                const S2 ph = phase(i, j);
                const T c = (T)ph.x, s = (T)ph.y;
                const T term = selfc ? gpr * c : (T)2 * (gpr * c - gpi * s);
                const T r = dres[idx] - term;
                dres[idx] = r;
                if (i < M && j < N) el += (double)dw[i * N + j] * (double)r * (double)r;
            }
            for (int off = 16; off; off >>= 1) el += __shfl_xor_sync(0xffffffffu, el, off);
            if (lane == 0) red[warp] = el;
            __syncthreads();
            if (t == 0) {
                double s = 0.0;
                for (int w = 0; w < NW; ++w) s += red[w];
                reinterpret_cast<T *>(A.energies)[(size_t)blockIdx.x * (I + 1) + it + 1] = (T)s;
            }
        }

        if (it + 1 == I) break;  // the last update is never observed

        // ---- (3) spectrum update by the shifted weight spectrum + next local argmax
        T best = (T)-1;
        int bj = -1;
        if constexpr (CF > 0) {
            const int cm = (vfix - b) & (CF - 1), cp = (vfix + b) & (CF - 1);
            if (selfc) {
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    const int u = u0 + C::RPR * j;
                    if (u < R1) {
                        const T2 lo = Wat((u - a) & (CF - 1), cm);
                        g_re[j] = fma(-gpr, lo.x, g_re[j]);
                        g_im[j] = fma(-gpr, lo.y, g_im[j]);
                        const T e = g_re[j] * g_re[j] + g_im[j] * g_im[j];
                        if (e > best) { best = e; bj = j; }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    const int u = u0 + C::RPR * j;
                    if (u < R1) {
                        const T2 lo = Wat((u - a) & (CF - 1), cm);
                        const T2 hi = Wat((u + a) & (CF - 1), cp);
                        const T sA = lo.x + hi.x, sB = lo.y - hi.y, sC = lo.y + hi.y, sD = lo.x - hi.x;
                        g_re[j] = fma(gpi, sB, fma(-gpr, sA, g_re[j]));
                        g_im[j] = fma(-gpi, sD, fma(-gpr, sC, g_im[j]));
                        const T e = g_re[j] * g_re[j] + g_im[j] * g_im[j];
                        if (e > best) { best = e; bj = j; }
                    }
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                if (gu[j] < R1) {
                    const int u = gu[j], v = gv[j];
                    int rm = u - a; if (rm < 0) rm += F1;
                    int cm = v - b; if (cm < 0) cm += F2;
                    const T2 lo = Wat(rm, cm);
                    if (selfc) {
                        g_re[j] = fma(-gpr, lo.x, g_re[j]);
                        g_im[j] = fma(-gpr, lo.y, g_im[j]);
                    } else {
                        int rp = u + a; if (rp >= F1) rp -= F1;
                        int cp = v + b; if (cp >= F2) cp -= F2;
                        const T2 hi = Wat(rp, cp);
                        const T sA = lo.x + hi.x, sB = lo.y - hi.y, sC = lo.y + hi.y, sD = lo.x - hi.x;
                        g_re[j] = fma(gpi, sB, fma(-gpr, sA, g_re[j]));
                        g_im[j] = fma(-gpi, sD, fma(-gpr, sC, g_im[j]));
                    }
                    const T e = g_re[j] * g_re[j] + g_im[j] * g_im[j];
                    if (e > best) { best = e; bj = j; }
                }
            }
        }
        key = 0ull;
        if (bj >= 0) {
            int lin2 = 0;
#pragma unroll
            for (int j = 0; j < NB; ++j)
                if (j == bj) lin2 = bin_u(j) * F2 + bin_v(j);
            key = pack_key(best, lin2);
        }
    }

    // ---- write-back of the block's LOST samples (conceal.py:61-66)
    if constexpr (MODE == 0) {
        T *img = reinterpret_cast<T *>(fd->image);
        for (int q = t; q < bh * bw; q += NT) {
            const int y = wr0 + br0 + q / bw, x = wc0 + bc0 + q % bw;
            if (fd->mask[(size_t)y * A.W + x] == FSE_LOST) img[(size_t)y * A.W + x] = model[q];
        }
    }
    if constexpr (DEBUG) {
        T *out = reinterpret_cast<T *>(A.residual) + (size_t)blockIdx.x * F1 * F2;
        __syncthreads();
        for (int idx = t; idx < F1 * F2; idx += NT) out[idx] = dres[idx];
    }
}

// ---------------------------------------------------------------------------
// Variant table and launch.

template <class C, int MODE, bool DEBUG>
int launch_variant(const KArgs &a, int grid, int Mmax, int Nmax, int F1max, int F2max, int model_n,
                   cudaStream_t s) {
    using T = typename C::T;
    const SmemLayout L = smem_layout<T, typename C::ST>(Mmax, Nmax, F1max, F2max, C::NW, model_n,
                                                        DEBUG, C::FULLW);
    int dev = 0, optin = 0;
    FSE_CUDA_TRY(cudaGetDevice(&dev));
    FSE_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (L.total > (size_t)optin)
        return fail(FSE_ENOTSUP, "window/FFT size needs " + std::to_string(L.total) +
                                     " B of shared memory (max " + std::to_string(optin) + ")");
    auto kern = fse_window_kernel<C, MODE, DEBUG>;
    FSE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    if (grid > 0) {
        kern<<<grid, C::NT, L.total, s>>>(a, L);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}


// Kernel variants: F=32/64/128 fast paths and the generic runtime-size path.
// NW (warps per CTA) per F: 6 / 6 / 20 -> NB = 3 / 11 / 13 bins per thread.
template <typename T> using CfgF32 = Cfg<T, T, 32, 6, true>;
template <typename T> using CfgF64 = Cfg<T, T, 64, 6, true>;
template <typename T> using CfgF128 = Cfg<T, T, 128, 20, std::is_same<T, float>::value>;
template <typename T> using CfgGen = Cfg<T, T, 0, 8, true>;

#define FSE_DECLARE_VARIANTS(EXT, T)                                                            \
    EXT template int launch_variant<CfgF32<T>, 0, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF64<T>, 0, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF128<T>, 0, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgGen<T>, 0, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF32<T>, 1, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF64<T>, 1, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF128<T>, 1, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgGen<T>, 1, false>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF32<T>, 1, true>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF64<T>, 1, true>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgF128<T>, 1, true>(const KArgs &, int, int, int, int, int, int, cudaStream_t); \
    EXT template int launch_variant<CfgGen<T>, 1, true>(const KArgs &, int, int, int, int, int, int, cudaStream_t);

FSE_DECLARE_VARIANTS(extern, float)
FSE_DECLARE_VARIANTS(extern, double)

}  // namespace fse
