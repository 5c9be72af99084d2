// FSE window kernel for ANY DFT size F1 x F2 (per window), sm_100a: the
// reference's own semantics, DFT = window shape (fse.py:158-159,
// _kernel.pyx:143-150), i.e. the drop-in call conceal(image, mask) with the
// default FseParams (B=16, d=16: 48x48 windows, clipped to 24..48 rows or
// columns on image borders), plus non-power-of-two fft_size.
//
// Same algorithm and data flow as the power-of-two kernel (fse_fast.cuh):
//   * g of the canonical half spectrum in registers (rows 0 .. F1/2, rows 0
//     and F1/2 only for v <= F2/2: one bin of each conjugate pair, the
//     reference's canonical picks, tests/reference.py:59-71), bins spread
//     linearly over the CTA (i = t + NT j), NB per thread;
//   * W in shared memory as a row-extended plane (rows -H .. 2H, H = F1/2), so
//     both shifted rows u -+ a are in range; columns wrap mod F2 with one
//     select each (F2 is a runtime value);
//   * tracked argmax: per-thread best (|g|^2, bin), warp REDUX + ballot, one
//     barrier, first maximum in row-major order (_kernel.pyx:32-44);
//   * p = g / sum(w) (_kernel.pyx:46-47) with sum(w) = W[0][0];
//     update g -= gamma (p W[k-j] + conj(p) W[k+j]) (_kernel.pyx:65-97), the
//     self-conjugate case as the general one with p halved and real (:50-64);
//   * the block model 2 Re(gamma p e^{+j 2 pi (a i / F1 + b j / F2)}) summed per
//     iteration by the thread of each block sample (fse.py:159 restricted to
//     the block), then the LOST samples written back (conceal.py:61-66).
// The DFT set-up is a direct separable DFT (column pass over the M rows of
// the window, row pass over the owned bins and the W half rows).
#pragma once

#include "fse_fast.cuh"

namespace fse {

template <typename T_, int NW_, int NB_, int MINB_ = 0>
struct GenCfg {
    using T = T_;
    using T2 = typename V2<T_>::type;
    static constexpr int NW = NW_;
    static constexpr int NT = NW_ * 32;
    static constexpr int NB = NB_;      // canonical bins per thread
    static constexpr int MINB = MINB_;  // __launch_bounds__ min blocks per SM
};

constexpr int GEN_WPT = 8;  // W half-plane outputs per thread (one round)

struct GenLayout {
    size_t tw1, tw2, slots, model, hist, big, yx, yw, xs, ws, total;
};

// Shared memory: twiddles, argmax slots, the block model, then one region
// used in turn for the staging tiles + column spectra and for the W plane.
template <typename T>
__host__ __device__ inline GenLayout gen_layout(int F1, int F2, int Mmax, int Nmax, int NW, int model_n,
                                                int iters) {
    GenLayout L;
    const size_t c2 = 2 * sizeof(T);
    auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t o = 0;
    L.tw1 = o; o = a16(o + (size_t)F1 * c2);
    L.tw2 = o; o = a16(o + (size_t)F2 * c2);
    L.slots = o; o = a16(o + 2 * (size_t)NW * sizeof(ArgSlot<double>));
    L.model = o; o = a16(o + (size_t)(model_n > 0 ? model_n : 1) * sizeof(T));
    L.hist = o; o = a16(o + (size_t)(iters > 0 ? iters : 1) * sizeof(PickRec<T>));
    o = (o + 127) & ~size_t(127);
    L.big = o;
    const size_t H = (size_t)F1 / 2;
    const size_t wext = (3 * H + 1) * (size_t)F2 * c2;
    const size_t yb = a16((H + 1) * (size_t)Nmax * c2);
    const size_t xb = a16((size_t)Mmax * Nmax * sizeof(T));
    // column pass: xs/ws -> Yx/Yw (separate); the W plane overwrites all four
    // once the row passes are done (its values are staged in registers first)
    L.yx = 0;
    L.yw = yb;
    L.xs = 2 * yb;
    L.ws = 2 * yb + xb;
    const size_t stage = 2 * yb + 2 * xb;
    L.total = L.big + (stage > wext ? stage : wext);
    return L;
}

// x mod m for 0 <= x < m * m (m <= 65535) without an integer division
__device__ __forceinline__ int small_mod(int x, int m, float inv_m) {
    int q = __float2int_rz((float)x * inv_m);
    int r = x - q * m;
    r += r < 0 ? m : 0;
    r -= r >= m ? m : 0;
    return r;
}

template <class C, int MODE, typename IT>
__device__ __forceinline__ void gen_window(const KArgs &A, const GenLayout &L, unsigned char *sm) {
    using T = typename C::T;
    using T2 = typename C::T2;
    constexpr int NT = C::NT, NW = C::NW, NB = C::NB;
    constexpr bool IS_F32 = sizeof(T) == 4;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    // ---- window geometry (grid.py:108-135)
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
    const int H = F1 / 2;
    const float inv1 = 1.0f / (float)F1, inv2 = 1.0f / (float)F2;

    T2 *tw1 = reinterpret_cast<T2 *>(sm + L.tw1);
    T2 *tw2 = reinterpret_cast<T2 *>(sm + L.tw2);
    ArgSlot<T> *slots = reinterpret_cast<ArgSlot<T> *>(sm + L.slots);
    T *model = reinterpret_cast<T *>(sm + L.model);
    PickRec<T> *hist = reinterpret_cast<PickRec<T> *>(sm + L.hist);
    unsigned char *big = sm + L.big;
    T2 *Yx = reinterpret_cast<T2 *>(big + L.yx);
    T2 *Yw = reinterpret_cast<T2 *>(big + L.yw);
    T *xs = reinterpret_cast<T *>(big + L.xs);
    T *ws = reinterpret_cast<T *>(big + L.ws);
    T2 *Wp = reinterpret_cast<T2 *>(big);  // ext row e = W row e - H, stride F2

    for (int k = t; k < F1; k += NT) {
        double s, c;
        sincospi(2.0 * k / F1, &s, &c);
        tw1[k] = T2{(T)c, (T)s};
    }
    for (int k = t; k < F2; k += NT) {
        double s, c;
        sincospi(2.0 * k / F2, &s, &c);
        tw2[k] = T2{(T)c, (T)s};
    }

    // ---- staging: classes -> weights (fse.py:105-119); x = w * select(w > 0, v, 0)
    if constexpr (MODE == 0) {
        const int myrank = fd->rank[blk];
        const IT *img = reinterpret_cast<const IT *>(fd->image);
        for (int idx = t; idx < M * N; idx += NT) {
            const int i = idx / N, j = idx - i * N;
            const int y = wr0 + i, x = wc0 + j;
            const size_t off = (size_t)y * A.W + x;
            const uint8_t s = fd->mask[off];
            const double dec = A.decay[abs(2 * i - (M - 1)) * A.decay_dim + abs(2 * j - (N - 1))];
            double w;
            if (s == FSE_LOST) {
                const int owner = (y / A.B) * A.cols + x / A.B;
                // R iff the owner block was written by an earlier batch
                // (snapshot semantics, conceal.py:148-163); BI/BO otherwise
                w = (owner != blk && fd->rank[owner] < myrank) ? A.delta * dec : 0.0;
            } else if (s == FSE_RECONSTRUCTED) {
                w = A.delta * dec;
            } else {
                w = dec;
            }
            const double v = (double)img[off];
            xs[idx] = w > 0.0 ? (T)(w * v) : (T)0;
            ws[idx] = (T)w;
        }
        for (int q = t; q < bh * bw; q += NT) model[q] = (T)0;
    } else {
        const T *val = reinterpret_cast<const T *>(A.values) + (size_t)blockIdx.x * M * N;
        const T *wgt = reinterpret_cast<const T *>(A.weights) + (size_t)blockIdx.x * M * N;
        for (int idx = t; idx < M * N; idx += NT) {
            const double w = (double)wgt[idx];
            const double r0 = w > 0.0 ? (double)val[idx] : 0.0;
            xs[idx] = (T)(w * r0);
            ws[idx] = (T)w;
        }
    }
    __syncthreads();

    // ---- DFT pass 1 (columns): Y[k1][n] = sum_m x[m][n] e^{-j 2 pi k1 m / F1}, k1 <= H
    for (int o = t; o < (H + 1) * N; o += NT) {
        const int k1 = o / N, n = o - k1 * N;
        T2 ax = T2{0, 0}, aw = T2{0, 0};
        int k = 0;
        for (int m = 0; m < M; ++m) {
            const T2 tw = tw1[k];
            const T xv = xs[m * N + n], wv = ws[m * N + n];
            ax = cfma(T2{xv, -xv}, tw, ax);
            aw = cfma(T2{wv, -wv}, tw, aw);
            k += k1;
            k -= k >= F1 ? F1 : 0;
        }
        Yx[o] = ax;
        Yw[o] = aw;
    }
    __syncthreads();

    // ---- canonical bins of this thread: i = t + NT j over rows 0 .. H in
    // row-major order (row 0 and, for even F1, row H: v <= F2/2 only)
    const int n0 = F2 / 2 + 1, Hf = (F1 - 1) / 2;
    const int nbins = n0 + Hf * F2 + ((F1 % 2 == 0 && F1 >= 2) ? n0 : 0);
    int bu[NB], bv[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        int i = t + NT * j, u = -1, v = 0;
        if (i < nbins) {
            if (i < n0) {
                u = 0;
                v = i;
            } else if ((i -= n0) < Hf * F2) {
                u = 1 + i / F2;
                v = i - (u - 1) * F2;
            } else {
                u = H;
                v = i - Hf * F2;
            }
        }
        bu[j] = u;
        bv[j] = v;
    }
    int uF2[NB];  // row offset of each bin in the W plane
#pragma unroll
    for (int j = 0; j < NB; ++j) uF2[j] = bu[j] * F2;
    auto row_dft = [&](const T2 *Y, int u, int v) -> T2 {  // sum_n Y[u][n] e^{-j 2 pi v n / F2}
        const T2 *yr = Y + u * N;
        T2 acc = T2{0, 0};
        int k = 0;
        for (int n = 0; n < N; ++n) {
            acc = dft_mac(acc, yr[n], tw2[k]);
            k += v;
            k -= k >= F2 ? F2 : 0;
        }
        return acc;
    };
    T2 G[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) G[j] = bu[j] >= 0 ? row_dft(Yx, bu[j], bv[j]) : T2{0, 0};
    // W half rows 0 .. H, all columns: values to registers (at most WPT per
    // thread, checked by the launcher), then -- after the barrier that retires
    // Yx/Yw/xs/ws, whose bytes the plane reuses -- into ext rows H .. 2H
    constexpr int WPT = GEN_WPT;
    const int nw = (H + 1) * F2;
    T2 wv[WPT];
#pragma unroll
    for (int r = 0; r < WPT; ++r) {
        const int o = t + NT * r;
        if (o < nw) {
            const int u = o / F2;
            wv[r] = row_dft(Yw, u, o - u * F2);
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < WPT; ++r) {
        const int o = t + NT * r;
        if (o < nw) Wp[(size_t)H * F2 + o] = wv[r];
    }
    __syncthreads();
    // the other rows by symmetry: W[r][c] = conj W[-r][-c]; W rows -H..-1 at
    // ext rows 0..H-1 and rows H+1..2H at ext rows 2H+1..3H
    for (int o = t; o < 2 * H * F2; o += NT) {
        const int q = o / F2, c = o - q * F2;
        const int r = q < H ? q - H : q + 1;  // W row
        const int src = r < 0 ? -r : F1 - r;  // in 0 .. H
        const T2 s = Wp[(size_t)(H + src) * F2 + (c == 0 ? 0 : F2 - c)];
        Wp[(size_t)(H + r) * F2 + c] = T2{s.x, -s.y};
    }
    __syncthreads();

    // sum(w) = W[0][0] (exact fp sums of the column/row passes, fixed order)
    const double total = (double)Wp[(size_t)H * F2].x;
    const T gamma = (T)A.gamma;
    const T tot = (T)total;
    const T inv_tot = (T)1 / tot;
    const T ginv = gamma * inv_tot;
    const int I = A.iterations;
    int32_t *picks_out = nullptr;
    T *plog = nullptr;
    if constexpr (MODE == 0) {
        if (A.picks) picks_out = A.picks + ((size_t)frame * A.rows * A.cols + blk) * (size_t)I * 2;
    } else {
        picks_out = A.picks + (size_t)blockIdx.x * I * 2;
        plog = reinterpret_cast<T *>(A.plog) + (size_t)blockIdx.x * I * 2;
    }
    const int nsamp = bh * bw;

    // ---- tracked argmax state
    T best = (T)0;
    unsigned blin = 0xFFFFFFFFu;
    T2 bg = T2{0, 0};
    auto track_all = [&]() {
        best = (T)0;
        blin = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const T e = energy(G[j]);
            if (bu[j] >= 0 && e > best) {
                best = e;
                blin = ((unsigned)bu[j] << 16) | (unsigned)bv[j];
                bg = G[j];
            }
        }
    };
    track_all();

    for (int it = 0; it < I; ++it) {
        ArgSlot<T> *asl = slots + (it & 1) * NW;
        const auto key = energy_key(best);
        if (lane == warp_argmax_lane(key, blin)) {
            ArgSlot<T> mine;
            mine.key = key;
            mine.lin = blin;
            mine.gre = bg.x;
            mine.gim = bg.y;
            asl[warp] = mine;
        }
        __syncthreads();
        const bool in = lane < NW;
        const auto uk = in ? asl[lane].key : decltype(asl[0].key)(0);
        const unsigned ul = in ? asl[lane].lin : 0xFFFFFFFFu;
        const int gw = warp_argmax_lane(uk, ul);
        unsigned glin = __shfl_sync(0xffffffffu, ul, gw);
        // no bin above 0 (all energies 0 or NaN): the reference's strict-'>'
        // scan from -1 keeps (0, 0) (_kernel.pyx:32-44), whose g is 0
        if (glin == 0xFFFFFFFFu) glin = 0;
        // bins are tagged (u << 16) | v: row-major order without a division
        const int a = (int)(glin >> 16), b = (int)(glin & 0xFFFFu);
        const T2 gwin = T2{asl[gw].gre, asl[gw].gim};
        // p = g / sum(w) (_kernel.pyx:46-47) with gamma / sum(w) folded into
        // one factor, as in the power-of-two kernel (fse_fast.cuh)
        T gpr = gwin.x * ginv, gpi = gwin.y * ginv;
        if (t == 0 && picks_out) {
            picks_out[2 * it] = a;
            picks_out[2 * it + 1] = b;
            if (plog) {
                if constexpr (IS_F32) {
                    plog[2 * it] = gwin.x * inv_tot;
                    plog[2 * it + 1] = gwin.y * inv_tot;
                } else {
                    plog[2 * it] = div_by(gwin.x, tot, inv_tot);
                    plog[2 * it + 1] = div_by(gwin.y, tot, inv_tot);
                }
            }
        }
        // self-conjugate: gamma Re(p) W[k - j] == (gamma Re(p) / 2)(W[k-j] + W[k+j])
        // (canonical picks have 0 <= a <= F1/2 and 0 <= b < F2)
        const bool selfc = (a == 0 || 2 * a == F1) && (b == 0 || 2 * b == F2);
        if (selfc) {
            gpr = gpr * (T)0.5;
            gpi = (T)0;
        }
        // the pick for the block model, synthesised after the loop
        if constexpr (MODE == 0) {
            if (t == 0) hist[it] = PickRec<T>{a, b, gpr, gpi};
        }
        if (it + 1 == I) break;  // the last spectrum update is never observed

        // ---- spectrum update by the shifted weight spectrum + next local argmax
        const T2 *rowlo = Wp + (size_t)(H - a) * F2;  // ext row of W row u - a is u - a + H
        const T2 *rowhi = Wp + (size_t)(H + a) * F2;
        best = (T)0;
        blin = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            if (bu[j] >= 0) {
                const int v = bv[j];
                int cm = v - b;
                cm += cm < 0 ? F2 : 0;
                int cp = v + b;
                cp -= cp >= F2 ? F2 : 0;
                const T2 lo = rowlo[uF2[j] + cm], hi = rowhi[uF2[j] + cp];
                if constexpr (IS_F32) G[j] = spectral_update_bc(G[j], lo, hi, -gpr, gpi);
                else G[j] = spectral_update(G[j], lo, hi, T2{-gpr, -gpr}, T2{gpi, -gpi});
                const T e = energy(G[j]);
                if (e > best) {
                    best = e;
                    blin = ((unsigned)bu[j] << 16) | (unsigned)v;
                    bg = G[j];
                }
            }
        }
    }

    // ---- block model 2 Re(gamma p e^{+j 2 pi (a i / F1 + b j / F2)}) summed in
    // iteration order (fse.py:159 restricted to the block), then the write-back
    // of the block's LOST samples (conceal.py:61-66)
    if constexpr (MODE == 0) {
        __syncthreads();
        IT *img = reinterpret_cast<IT *>(fd->image);
        for (int q = t; q < nsamp; q += NT) {
            const int mi = br0 + q / bw, mj = bc0 + q % bw;
            T acc = (T)0;
            for (int it = 0; it < I; ++it) {
                const PickRec<T> h = hist[it];
                const T2 p1 = tw1[small_mod(h.a * mi, F1, inv1)], p2 = tw2[small_mod(h.b * mj, F2, inv2)];
                const T c = p1.x * p2.x - p1.y * p2.y, sn = p1.x * p2.y + p1.y * p2.x;
                acc += (T)2 * (h.gpr * c - h.gpi * sn);
            }
            const size_t off = (size_t)(wr0 + br0 + q / bw) * A.W + (wc0 + bc0 + q % bw);
            if (fd->mask[off] == FSE_LOST) img[off] = (IT)acc;
        }
    }
}

template <class C, int MODE>
__global__ void __launch_bounds__(C::NT, C::MINB) fse_gen_kernel(const KArgs A, const GenLayout L) {
    extern __shared__ __align__(128) unsigned char sm[];
    gen_window<C, MODE, typename C::T>(A, L, sm);
}

// Host launcher (fse_inst_gen.cu): FSE_ENOTSUP when the sizes do not fit.
int gen_launch(int dtype, int mode, const KArgs &a, int grid, int Mmax, int Nmax, int F1max, int F2max,
               int model_n, cudaStream_t s);

}  // namespace fse
