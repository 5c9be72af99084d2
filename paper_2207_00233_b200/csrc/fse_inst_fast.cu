// Instantiation + host launchers of the fast-path kernel (fse_fast.cuh).
#include <atomic>
#include <cstdlib>
#include <algorithm>
#include <string>
#include <type_traits>

#include "fse_fast.cuh"

namespace fse {

// Per-device launch state.  cudaFuncSetAttribute applies to the current
// device only, so the "largest dynamic shared memory configured" record of
// each kernel is kept per device (a process may drive several GPUs), and so
// is the SM count.
constexpr int kMaxDev = 64;
static int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return dev;
}
static int device_sms(int dev) {
    static std::atomic<int> cache[kMaxDev] = {};
    if (dev < 0 || dev >= kMaxDev) dev = 0;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 148;
        }
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}
// Raise kern's dynamic shared-memory limit on the current device to `bytes`
// (once per kernel, device and size).  Tag: one static per kernel instance.
template <class... K> struct KTag {};  // one type per kernel instance
template <class Tag>
static int ensure_smem(const void *kern, size_t bytes) {
    static std::atomic<size_t> configured[kMaxDev] = {};
    const int dev = current_device();
    std::atomic<size_t> &c = configured[dev < kMaxDev ? dev : 0];
    if (bytes <= c.load(std::memory_order_acquire)) return FSE_OK;
    int optin = 0;
    FSE_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (bytes > (size_t)optin)
        return fail(FSE_ENOTSUP, "fast kernel needs " + std::to_string(bytes) + " B of shared memory");
    FSE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    size_t cur = c.load(std::memory_order_relaxed);
    while (bytes > cur && !c.compare_exchange_weak(cur, bytes)) {
    }
    return FSE_OK;
}

// F = 64: 66 row segments of the half plane over 6 warps -> 11 bins per thread
// (4 warps / 17 bins measured 5% slower: fewer warps to hide latency).
// F = 32: 17 row segments over 6 warps -> 3 bins per thread.
// min blocks/SM in __launch_bounds__ pins the register budget to the occupancy
// the shared memory allows (an explicit 1 lets ptxas take 121 registers and
// halves the fp32 occupancy)
#ifndef FSE_F64_NW  // dev knob: warps per window of the wide fp64 F = 64 kernel
#define FSE_F64_NW 6
#endif
template <typename T>
using Fast64 = FastCfg<T, 64, sizeof(T) == 4 ? 6 : FSE_F64_NW, sizeof(T) == 4, sizeof(T) == 4 ? 4 : 3>;  // fp64: plain W plane

// F = 32 fp32: 3 warps per window (6 bins per thread), 8 CTAs per SM --
// config 5 B=2 (1.04M windows of 30x30): 95 ms vs 120 ms with 6 warps
// (measured NW/MINB: 6/0 120, 3/10 98, 3/6 104, 2/12 99, 2/16 109, 1/16 115 ms)
#ifndef FSE_F32_32_NW  // dev knob
#define FSE_F32_32_NW 3
#define FSE_F32_32_MINB 8
#endif
// fp64 F = 32: 3 warps per window (6 bins per thread) at >= 6 CTAs per SM --
// config 5 B=2 fp64 (922 levels, 1.04M windows) 178.1 -> 160.5 ms device
// (6 warps: 178.1; 3 warps at 8 CTAs/SM, 80 registers: 170.1)
#ifndef FSE_F64_32_NW  // dev knobs: the fp64 F = 32 kernel
#define FSE_F64_32_NW 3
#define FSE_F64_32_MINB 6
#endif
template <typename T>
using Fast32 = FastCfg<T, 32, sizeof(T) == 4 ? FSE_F32_32_NW : FSE_F64_32_NW, true,
                       sizeof(T) == 4 ? FSE_F32_32_MINB : FSE_F64_32_MINB>;
// tracked-argmax fp32 twins for narrow levels (see FastCfg::TRACK)
using Fast64T = FastCfg<float, 64, 6, true, 4, 1, true>;
// levels of at most one window per SM (config 2; config 5 bands at N = 8):
// 12 warps per window (6 bins per thread) shorten a lone window's iteration --
// config 2 5.3 -> 5.0 ms; with more windows per level the 6-warp form wins
// (config 3: 19.8 vs 23.3 ms; 22 warps: slower everywhere)
#ifndef FSE_NARROW_LG  // dev knob: gather group of the narrow-level variants
#define FSE_NARROW_LG 0
#endif
#ifndef FSE_NARROW_MINB
#define FSE_NARROW_MINB 2
#endif
using Fast64L = FastCfg<float, 64, 12, true, FSE_NARROW_MINB, 1, true, FSE_NARROW_LG>;
using Fast32T = FastCfg<float, 32, FSE_F32_32_NW, true, FSE_F32_32_MINB, 1, true>;
// fp64 levels of at most one window per SM (configs 1 and 2, narrow levels of
// 3 and 5) with 12 warps per window: a lone window's set-up drops from 40 to
// 20 us (the 6-warp kernel spills at its 3-CTA register cap), the iteration
// stays at ~0.7 us (the W gathers bound it); config 1 1.90 -> 1.86 ms, config 2
// 8.35 -> 8.13 ms (22 warps: 2.02 / 9.05 ms).  FSE_F64L = 0 / 22 selects the
// 6-warp kernel / the 22-warp variant instead.
// (gathers in groups of 3 bins: a lone window's update loop 971 -> 926 cycles
// per iteration, profiles/r2/narrow_lg_ab_r2h.jsonl)
using Fast64D12 = FastCfg<double, 64, 12, false, 1, 1, false, FSE_NARROW_LG ? FSE_NARROW_LG : 3>;
using Fast64D22 = FastCfg<double, 64, 22, false, 1>;
static int f64_narrow_warps() {
    static const int v = [] {
        const char *e = getenv("FSE_F64L");
        return e ? atoi(e) : 12;
    }();
    return v;
}

// Levels narrower than this many windows use the tracked argmax (fp32):
// measured on configs 2 (linescan), 3 and 5 -- levels of a few hundred
// windows -- 3-10% faster, on config 4's levels of thousands 1% slower.
// Default 16 x SMs; FSE_TRACK_BELOW or fse_set_track_below override (0 = never).
// Both forms compute the same argmax, so results are identical.
std::atomic<int> g_track_below{-1};
static int track_below(int sms) {
    int v = g_track_below.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = getenv("FSE_TRACK_BELOW");
        v = e ? atoi(e) : 16 * sms;
        int expect = -1;
        g_track_below.compare_exchange_strong(expect, v);
        v = g_track_below.load(std::memory_order_relaxed);
    }
    return v;
}
// F = 128 (fp32 only: the row-extended W plane is 193 x 128 x 8 B = 198 KB):
// 260 row segments over 20 warps -> 13 bins per thread, one CTA per SM.
#ifndef FSE_F128_NW  // dev knob: warps per window of the fp32 F = 128 kernel
#define FSE_F128_NW 20
#endif
template <typename T> using Fast128 = FastCfg<T, 128, FSE_F128_NW>;
#ifndef FSE_F128T_NW
#define FSE_F128T_NW FSE_F128_NW
#endif
using Fast128T = FastCfg<float, 128, FSE_F128T_NW, true, 0, 1, true>;
#ifdef FSE_WITH_CLUSTER  // experiment, measured slower everywhere: not in the default build
// Cluster variants for levels narrower than the GPU: one window over CL SMs.
#ifndef FSE_CL_NW  // dev knob: warps per CTA of the F = 64 cluster variants
#define FSE_CL_NW 6
#endif
template <typename T, int CL> using Fast64C = FastCfg<T, 64, (FSE_CL_NW < 32 / CL ? FSE_CL_NW : 32 / CL), sizeof(T) == 4, 0, CL>;
template <typename T, int CL> using Fast32C = FastCfg<T, 32, 6, true, 0, CL>;

// FSE_CLUSTER: unset / 0 = off (default), 2 / 4 = that cluster size, -1 = automatic.
// Off by default: measured slower than one CTA per window even on the narrow
// levels of configs 1, 2 and 5 (the per-iteration cluster barrier costs more
// than the shorter bin loop saves).
static int cluster_mode() {
    static int v = [] {
        const char *e = getenv("FSE_CLUSTER");
        return e ? atoi(e) : 0;
    }();
    return v;
}
bool cluster_levels() { return cluster_mode() != 0; }

template <class C>
static int launch_cluster(const FastArgs &a, int windows, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    const FastLayout L = fast_layout<typename C::T>(C::F, C::NWT, Mmax, Nmax, model_n, a.iterations, C::HALF ? 2 : (C::EXT ? 1 : 0));
    auto kern = fse_fast_cluster_kernel<C>;
    if (int rc = ensure_smem<KTag<C, std::integral_constant<int, 100>>>((const void *)kern, L.total)) return rc;
    if (windows > 0) {
        kern<<<windows * C::CL, C::NT, L.total, s>>>(a, L);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}
#else
bool cluster_levels() { return false; }
#endif
// (A 22-warp / 3-bin "latency" variant for levels narrower than the GPU was
// measured 20% slower on configs 1-2: per-iteration overhead grows with warps.)

// F = 128 fp64: half-plane W (65 x 128 x 16 B = 133 KB, the w-combine in
// place over the partials), 20 warps (13 bins per thread), one CTA per SM.
#ifndef FSE_F128D_LG
#define FSE_F128D_LG 0
#endif
using Fast128D = FastCfg<double, 128, 20, 2, 1, 1, false, FSE_F128D_LG>;

int fast_supported(int dtype, int F, int Mmax, int Nmax, int model_n, int iterations) {
    // model samples live in registers: at most 2 per thread
    bool sizes = F == 32 || F == 64 || F == 128;
#ifdef FSE_NO_F128_F64  // dev A/B: fp64 F = 128 on the generic kernel, as before the half plane
    if (F == 128 && dtype == FSE_F64) return 0;
#endif
    if (F == 128 && dtype == FSE_F64) {
        // the half plane leaves room for windows up to ~40 x 40 (B = 8, d <= 16)
        const FastLayout L = fast_layout<double>(128, Fast128D::NWT, Mmax, Nmax, model_n, iterations, 2);
        sizes = L.total <= (size_t)227 * 1024;
    }
    return sizes && Mmax <= F && Nmax <= F && model_n <= 2 * 6 * 32;
}

// Level launches with programmatic dependent launch (FSE_PDL=1; the kernel
// waits for the previous grid in the stream before any global access).  Off by
// default: measured slower -- config 1 1.86 vs 1.80 ms, config 2 fp32 5.96 vs
// 5.30 ms, config 5 B=2 fp64 163.9 vs 160.8 ms (the next level's early CTAs
// hold SM slots while they wait); only config 2 fp64 gained (7.69 vs 7.81 ms).
static bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("FSE_PDL");
        return e && atoi(e) != 0;
    }();
    return on;
}

template <class C, int MODE, bool GUARD, bool TWIN = false>
static int launch_as(const FastArgs &a, int grid, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    FastLayout L = fast_layout<typename C::T>(C::F, C::NWT, Mmax, Nmax, model_n, a.iterations, C::HALF ? 2 : (C::EXT ? 1 : 0));
#ifdef FSE_SMEM_PAD
    L.total += FSE_SMEM_PAD;  // dev: occupancy sensitivity experiments
#endif
    auto kern = fse_fast_kernel<C, MODE, GUARD, TWIN>;
    if (int rc = ensure_smem<KTag<C, std::integral_constant<int, MODE>, std::integral_constant<bool, GUARD>, std::integral_constant<bool, TWIN>>>((const void *)kern, L.total)) return rc;
    if (grid > 0) {
        if (pdl_enabled()) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(C::NT);
            cfg.dynamicSmemBytes = L.total;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            FSE_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, L));
        } else {
            kern<<<grid, C::NT, L.total, s>>>(a, L);
        }
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}

// Level launches of a session with a weight-spectrum cache (a.wslot set) use
// the instance that also holds the cached-W path.
template <class C, int MODE, bool GUARD>
static int launch(const FastArgs &a, int grid, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    if constexpr (MODE == 0 && !GUARD && C::CL == 1) {
        if (a.wslot) return launch_as<C, MODE, GUARD, true>(a, grid, Mmax, Nmax, model_n, s);
    }
    return launch_as<C, MODE, GUARD, false>(a, grid, Mmax, Nmax, model_n, s);
}

template <class C>
static int launch_redo(const FastArgs &a, int max_entries, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    const FastLayout L = fast_layout<typename C::T>(C::F, C::NWT, Mmax, Nmax, model_n, a.iterations, C::HALF ? 2 : (C::EXT ? 1 : 0));
    auto kern = fse_fast_redo_kernel<C, float>;
    if (int rc = ensure_smem<KTag<C, std::integral_constant<int, 101>>>((const void *)kern, L.total)) return rc;
    int per_sm = 0;
    const int sms = device_sms(current_device());
    FSE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, L.total));
    int grid = std::min(max_entries, std::max(1, per_sm) * std::max(1, sms));
    if (grid > 0) {
        kern<<<grid, C::NT, L.total, s>>>(a, L);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FSE_OK;
}

template <class C, typename IT>
static int launch_dataflow(const FastArgs &a, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    const FastLayout L = fast_layout<typename C::T>(C::F, C::NWT, Mmax, Nmax, model_n, a.iterations, C::HALF ? 2 : (C::EXT ? 1 : 0));
    auto kern = fse_fast_dataflow_kernel<C, IT>;
    if (int rc = ensure_smem<KTag<C, IT, std::integral_constant<int, 102>>>((const void *)kern, L.total)) return rc;
    int per_sm = 0;
    const int sms = device_sms(current_device());
    FSE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, L.total));
    if (per_sm < 1) return fail(FSE_ENOTSUP, "dataflow kernel does not fit on an SM");
    const int grid = std::max(1, std::min(a.total, per_sm * sms));
    {
        const int ib = 256, ig = std::max(1, std::min((a.total + ib - 1) / ib, sms * 8));
        dataflow_init_kernel<<<ig, ib, 0, s>>>(a);
        FSE_CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    FastArgs args = a;
    FastLayout lay = L;
    void *params[] = {&args, &lay};
    // cooperative launch: the whole grid is co-resident (the dependency waits
    // rely on it)
    FSE_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(C::NT), params, L.total, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FSE_OK;
}

int fast_dataflow(int dtype, int F, const FastArgs &a, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    if (dtype == FSE_F32) {
        if (F == 128) return launch_dataflow<Fast128<float>, float>(a, Mmax, Nmax, model_n, s);
        if (F == 64) return launch_dataflow<Fast64<float>, float>(a, Mmax, Nmax, model_n, s);
        return launch_dataflow<Fast32<float>, float>(a, Mmax, Nmax, model_n, s);
    }
    if (F == 128) return launch_dataflow<Fast128D, double>(a, Mmax, Nmax, model_n, s);
    if (F == 64) return launch_dataflow<Fast64<double>, double>(a, Mmax, Nmax, model_n, s);
    return launch_dataflow<Fast32<double>, double>(a, Mmax, Nmax, model_n, s);
}

int fast_level(int dtype, int F, bool guard, const FastArgs &a, int grid, int Mmax, int Nmax,
               int model_n, cudaStream_t s) {
    const int sms = device_sms(current_device());
#ifdef FSE_WITH_CLUSTER
    // narrow level: give each window 4 (or 2) SMs as a cluster
    if (!guard && cluster_levels() && (F == 64 || F == 32) && grid * 2 <= sms) {
        const bool four = cluster_mode() == 4 || (cluster_mode() != 2 && grid * 4 <= sms);
        if (dtype == FSE_F32) {
            if (F == 64)
                return four ? launch_cluster<Fast64C<float, 4>>(a, grid, Mmax, Nmax, model_n, s)
                            : launch_cluster<Fast64C<float, 2>>(a, grid, Mmax, Nmax, model_n, s);
            return four ? launch_cluster<Fast32C<float, 4>>(a, grid, Mmax, Nmax, model_n, s)
                        : launch_cluster<Fast32C<float, 2>>(a, grid, Mmax, Nmax, model_n, s);
        }
        if (F == 64)
            return four ? launch_cluster<Fast64C<double, 4>>(a, grid, Mmax, Nmax, model_n, s)
                        : launch_cluster<Fast64C<double, 2>>(a, grid, Mmax, Nmax, model_n, s);
        return four ? launch_cluster<Fast32C<double, 4>>(a, grid, Mmax, Nmax, model_n, s)
                    : launch_cluster<Fast32C<double, 2>>(a, grid, Mmax, Nmax, model_n, s);
    }
#endif
    if (dtype == FSE_F32) {
        const bool narrow = grid < track_below(sms);
        if (F == 128)
            return narrow ? launch<Fast128T, 0, false>(a, grid, Mmax, Nmax, model_n, s)
                          : launch<Fast128<float>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
        if (F == 64) {
            if (guard) return launch<Fast64<float>, 0, true>(a, grid, Mmax, Nmax, model_n, s);
            if (narrow && grid <= sms && track_below(sms) > 0)
                return launch<Fast64L, 0, false>(a, grid, Mmax, Nmax, model_n, s);
            return narrow ? launch<Fast64T, 0, false>(a, grid, Mmax, Nmax, model_n, s)
                          : launch<Fast64<float>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
        }
        if (guard) return launch<Fast32<float>, 0, true>(a, grid, Mmax, Nmax, model_n, s);
        return narrow ? launch<Fast32T, 0, false>(a, grid, Mmax, Nmax, model_n, s)
                      : launch<Fast32<float>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
    }
    if (F == 128) return launch<Fast128D, 0, false>(a, grid, Mmax, Nmax, model_n, s);
    if (F == 64) {
        if (grid <= sms && f64_narrow_warps() == 12) return launch<Fast64D12, 0, false>(a, grid, Mmax, Nmax, model_n, s);
        if (grid <= sms && f64_narrow_warps() == 22) return launch<Fast64D22, 0, false>(a, grid, Mmax, Nmax, model_n, s);
        return launch<Fast64<double>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
    }
    return launch<Fast32<double>, 0, false>(a, grid, Mmax, Nmax, model_n, s);
}

int fast_redo(int F, const FastArgs &a, int max_entries, int Mmax, int Nmax, int model_n, cudaStream_t s) {
    if (F == 64) return launch_redo<Fast64<double>>(a, max_entries, Mmax, Nmax, model_n, s);
    return launch_redo<Fast32<double>>(a, max_entries, Mmax, Nmax, model_n, s);
}

// One variant per (precision, F): every variant of one F forms W with the same
// operation order (the column pass sums over m, the row pass over n, whatever
// the warp count), so its planes serve all of them.
int fast_wplanes(int dtype, int F, const FastArgs &a, int grid, int Mmax, int Nmax, int model_n,
                 cudaStream_t s) {
    if (dtype == FSE_F32) {
        if (F == 128) return launch<Fast128<float>, 2, false>(a, grid, Mmax, Nmax, model_n, s);
        if (F == 64) return launch<Fast64<float>, 2, false>(a, grid, Mmax, Nmax, model_n, s);
        return launch<Fast32<float>, 2, false>(a, grid, Mmax, Nmax, model_n, s);
    }
    if (F == 128) return launch<Fast128D, 2, false>(a, grid, Mmax, Nmax, model_n, s);
    if (F == 64) return launch<Fast64<double>, 2, false>(a, grid, Mmax, Nmax, model_n, s);
    return launch<Fast32<double>, 2, false>(a, grid, Mmax, Nmax, model_n, s);
}

int fast_windows(int dtype, int F, const FastArgs &a, int grid, cudaStream_t s) {
    if (dtype == FSE_F32) {
        if (F == 128) return launch<Fast128<float>, 1, false>(a, grid, a.M, a.N, 0, s);
        if (F == 64) return launch<Fast64<float>, 1, false>(a, grid, a.M, a.N, 0, s);
        return launch<Fast32<float>, 1, false>(a, grid, a.M, a.N, 0, s);
    }
    if (F == 128) return launch<Fast128D, 1, false>(a, grid, a.M, a.N, 0, s);
    if (F == 64) return launch<Fast64<double>, 1, false>(a, grid, a.M, a.N, 0, s);
    return launch<Fast32<double>, 1, false>(a, grid, a.M, a.N, 0, s);
}

}  // namespace fse

#ifdef FSE_CLOCKS
extern "C" int fse_debug_clocks(long long *out, int n) {
    return cudaMemcpyFromSymbol(out, fse::g_fse_clk, sizeof(long long) * (size_t)std::min(n, 1032)) == cudaSuccess
               ? 0
               : -5;
}
#endif
