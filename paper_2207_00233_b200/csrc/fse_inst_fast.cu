// Instantiation + host launchers of the fast-path kernel (fse_fast.cuh).
#include <cstdlib>
#include <string>

#include "fse_fast.cuh"

namespace fse {

// F = 64: 66 row segments of the half plane over 6 warps -> 11 bins per thread
// (4 warps / 17 bins measured 5% slower: fewer warps to hide latency).
// F = 32: 17 row segments over 6 warps -> 3 bins per thread.
template <typename T> using Fast64 = FastCfg<T, 64, 6>;

template <typename T> using Fast32 = FastCfg<T, 32, 6>;

int fast_supported(int F, int Mmax, int Nmax, int model_n) {
    // model samples live in registers: at most 2 per thread
    return (F == 32 || F == 64) && Mmax <= F && Nmax <= F && model_n <= 2 * 6 * 32;
}

template <class C, int MODE, bool GUARD>
static int launch(const FastArgs &a, int grid, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    const FastLayout L = fast_layout<typename C::T>(C::F, C::NW, Mmax, Nmax, model_n, a.iterations);
    auto kern = fse_fast_kernel<C, MODE, GUARD>;
    static thread_local size_t configured = 0;  // largest dynamic smem size set so far
    if (L.total > configured) {
        int dev = 0, optin = 0;
        FSE_CUDA_TRY(cudaGetDevice(&dev));
        FSE_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (L.total > (size_t)optin)
            return fail(FSE_ENOTSUP, "fast kernel needs " + std::to_string(L.total) + " B of shared memory");
        FSE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
        configured = L.total;
    }
    if (grid > 0) {
        kern<<<grid, C::NT, L.total, s>>>(a, L);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}

template <class C>
static int launch_redo(const FastArgs &a, int max_entries, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    const FastLayout L = fast_layout<typename C::T>(C::F, C::NW, Mmax, Nmax, model_n, a.iterations);
    auto kern = fse_fast_redo_kernel<C, float>;
    static thread_local size_t configured = 0;
    static thread_local int per_sm = 0, sms = 0;
    if (L.total > configured) {
        int dev = 0;
        FSE_CUDA_TRY(cudaGetDevice(&dev));
        FSE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
        FSE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, L.total));
        FSE_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        configured = L.total;
    }
    int grid = std::min(max_entries, std::max(1, per_sm) * std::max(1, sms));
    if (grid > 0) {
        kern<<<grid, C::NT, L.total, s>>>(a, L);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}

int fast_level(int dtype, int F, bool guard, const FastArgs &a, int grid, int Mmax, int Nmax,
               int model_n, cudaStream_t s) {
    if (dtype == FSE_F32) {
        if (F == 64)
            return guard ? launch<Fast64<float>, 0, true>(a, grid, Mmax, Nmax, model_n, s)
                         : launch<Fast64<float>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
        return guard ? launch<Fast32<float>, 0, true>(a, grid, Mmax, Nmax, model_n, s)
                     : launch<Fast32<float>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
    }
    if (F == 64) return launch<Fast64<double>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
    return launch<Fast32<double>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
}

int fast_redo(int F, const FastArgs &a, int max_entries, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    if (F == 64) return launch_redo<Fast64<double>>(a, max_entries, Mmax, Nmax, model_n, s);
    return launch_redo<Fast32<double>>(a, max_entries, Mmax, Nmax, model_n, s);
}

int fast_windows(int dtype, int F, const FastArgs &a, int grid, cudaStream_t s) {
    if (dtype == FSE_F32) {
        if (F == 64) return launch<Fast64<float>, 1, false>(a, grid, a.M, a.N, 0, s);
        return launch<Fast32<float>, 1, false>(a, grid, a.M, a.N, 0, s);
    }
    if (F == 64) return launch<Fast64<double>, 1, false>(a, grid, a.M, a.N, 0, s);
    return launch<Fast32<double>, 1, false>(a, grid, a.M, a.N, 0, s);
}

}  // namespace fse
