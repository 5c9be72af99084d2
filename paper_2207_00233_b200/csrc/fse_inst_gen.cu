// Instantiation + host launcher of the any-size kernel (fse_gen.cuh).
#include <atomic>
#include <string>

#include "fse_gen.cuh"

namespace fse {

// 12 warps per window: the reference-default windows (48 x 48, 1154 canonical
// bins) sit one per SM on their dependency levels, so a window's latency, not
// the SM's throughput, sets the time; NB covers up to 384 * NB bins.
template <typename T, int NB> using Gen = GenCfg<T, 12, NB>;
// windows of up to 1,280 canonical bins (the reference default 48 x 48 has
// 1,154): 8 warps x 5 bins at two CTAs per SM, so a dependency level of up
// to 2 x SMs windows is one wave
#ifndef FSE_GEN_NARROW8
#define FSE_GEN_NARROW8 1
#endif
template <typename T> using Gen8 = GenCfg<T, 8, 5, 2>;

static int gen_dev() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return d;
}

template <class C, int MODE>
static int launch_gen(const KArgs &a, int grid, int Mmax, int Nmax, int F1max, int F2max, int model_n,
                      cudaStream_t s) {
    using T = typename C::T;
    const GenLayout L = gen_layout<T>(F1max, F2max, Mmax, Nmax, C::NW, model_n, a.iterations);
    auto kern = fse_gen_kernel<C, MODE>;
    static std::atomic<size_t> configured[64] = {};
    const int dev = gen_dev();
    std::atomic<size_t> &c = configured[dev < 64 ? dev : 0];
    if (L.total > c.load()) {
        int optin = 0;
        FSE_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (L.total > (size_t)optin) return fail(FSE_ENOTSUP, "any-size kernel: shared memory");
        FSE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
        size_t cur = c.load();
        while (L.total > cur && !c.compare_exchange_weak(cur, L.total)) {
        }
    }
    if (grid > 0) {
        kern<<<grid, C::NT, L.total, s>>>(a, L);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}

template <typename T, int MODE>
static int pick(const KArgs &a, int grid, int Mmax, int Nmax, int F1, int F2, int model_n, cudaStream_t s) {
    constexpr int NT = Gen<T, 4>::NT;
    // canonical bins of the largest DFT and W half-plane outputs per thread
    const long bins = (long)(F2 / 2 + 1) * (F1 % 2 == 0 ? 2 : 1) + (long)((F1 - 1) / 2) * F2;
    const long wout = (long)(F1 / 2 + 1) * F2;
    if (wout > (long)NT * GEN_WPT) return fail(FSE_ENOTSUP, "any-size kernel: W half plane too large");
    if (FSE_GEN_NARROW8 && bins <= 5L * Gen8<T>::NT && wout <= (long)Gen8<T>::NT * GEN_WPT)
        return launch_gen<Gen8<T>, MODE>(a, grid, Mmax, Nmax, F1, F2, model_n, s);
    if (bins <= 4L * NT) return launch_gen<Gen<T, 4>, MODE>(a, grid, Mmax, Nmax, F1, F2, model_n, s);
    if (bins <= 8L * NT) return launch_gen<Gen<T, 8>, MODE>(a, grid, Mmax, Nmax, F1, F2, model_n, s);
    return fail(FSE_ENOTSUP, "any-size kernel: too many bins");
}

int gen_launch(int dtype, int mode, const KArgs &a, int grid, int Mmax, int Nmax, int F1max, int F2max,
               int model_n, cudaStream_t s) {
    if (model_n > 4096) return fail(FSE_ENOTSUP, "any-size kernel: block too large");
    if (dtype == FSE_F64)
        return mode == 0 ? pick<double, 0>(a, grid, Mmax, Nmax, F1max, F2max, model_n, s)
                         : pick<double, 1>(a, grid, Mmax, Nmax, F1max, F2max, model_n, s);
    return mode == 0 ? pick<float, 0>(a, grid, Mmax, Nmax, F1max, F2max, model_n, s)
                     : pick<float, 1>(a, grid, Mmax, Nmax, F1max, F2max, model_n, s);
}

}  // namespace fse
