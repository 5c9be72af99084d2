// Device side of libfse_b200: the per-window operator entry point and the
// level-by-level concealment pipeline (host orchestration of the sm_100a
// kernel in fse_kernel.cuh).  See include/fse_b200.h for the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fse_fast.cuh"

namespace fse {

std::atomic<long long> g_launches{0};

// Optional device timing of the level launches (bench.py's roofline): one
// (start, stop) event pair per fse_conceal_frames call, recorded on its stream.
struct TimingState {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    long long window_launches = 0;
    // per-call guard counters copied back asynchronously (pinned), summed on read
    std::vector<std::pair<int *, int>> redo;
};
static thread_local TimingState g_timing;

// fp32 near-tie guard thresholds (fse_fast.cuh): redo in fp64 when
// e1 - e2 <= (tau0 + tau1 * it) * e1.  Negative tau0 disables the guard.
static double g_tau0 = -1.0, g_tau1 = 0.0;

// Persistent dataflow launch instead of one launch per level.  Off by default:
// measured on config 4 it ties the level launches (fp32) or loses 5% (fp64) —
// the critical path is the DAG depth either way and the level launches already
// keep ~97% wave efficiency.  FSE_DATAFLOW=1 or fse_set_dataflow(1) selects it.
static bool g_dataflow = [] {
    const char *e = getenv("FSE_DATAFLOW");
    return e && e[0] == '1';
}();
bool dataflow_enabled() { return g_dataflow; }
static long long g_redo_total = 0;

// FP32 FMA throughput probe: 8 independent FFMA chains per thread.
__global__ void fma_probe_kernel(float *out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

// FFMA2 (packed f32x2) and DFMA throughput probes: 8 independent chains.
__global__ void fma2_probe_kernel(float *out, int iters, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = cfma(make_float2(a, a), x[k], make_float2(b, b));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    if (s == 12345.678f) out[0] = s;
}
__global__ void dfma_probe_kernel(float *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = (float)s;
}

// LOST samples of concealed blocks become RECONSTRUCTED (conceal.py:65-66)
__global__ void finalize_masks_kernel(const FrameDesc *frames, int n, int H, int W, int B, int cols) {
    const long long total = (long long)n * H * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(i / ((long long)H * W));
        const long long p = i - (long long)f * H * W;
        const int y = (int)(p / W), x = (int)(p - (long long)y * W);
        const FrameDesc &fd = frames[f];
        uint8_t s = fd.mask[p];
        if (s == FSE_LOST && fd.rank[(y / B) * cols + x / B] != INT_MAX) s = FSE_RECONSTRUCTED;
        fd.mask_out[p] = s;
    }
}



template <typename T, int MODE, bool DEBUG>
int dispatch(const KArgs &a, int grid, int Mmax, int Nmax, int F1, int F2, int model_n,
             cudaStream_t s) {
    if (F1 == F2 && F1 >= Mmax && F2 >= Nmax) {
        if (F1 == 32) return launch_variant<CfgF32<T>, MODE, DEBUG>(a, grid, Mmax, Nmax, 32, 32, model_n, s);
        if (F1 == 64) return launch_variant<CfgF64<T>, MODE, DEBUG>(a, grid, Mmax, Nmax, 64, 64, model_n, s);
        if (F1 == 128) return launch_variant<CfgF128<T>, MODE, DEBUG>(a, grid, Mmax, Nmax, 128, 128, model_n, s);
    }
    const int F1m = F1 ? F1 : Mmax, F2m = F2 ? F2 : Nmax;
    if ((F1m / 2 + 1) * F2m > CfgGen<T>::NB * CfgGen<T>::NT)
        return fail(FSE_ENOTSUP, "DFT size " + std::to_string(F1m) + "x" + std::to_string(F2m) +
                                     " exceeds the generic kernel's bin capacity");
    return launch_variant<CfgGen<T>, MODE, DEBUG>(a, grid, Mmax, Nmax, F1m, F2m, model_n, s);
}

}  // namespace fse

using fse::fail;

extern "C" {

int fse_version(int32_t *out, int32_t n) {
    int32_t v[6] = {1, 3, 32, 64, 128, -1};
    int dev = 0, sms = -1;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
        v[5] = sms;
    else
        cudaGetLastError();
    for (int i = 0; i < n && i < 6; ++i) out[i] = v[i];
    return FSE_OK;
}

int fse_timing_enable(int32_t on) {
    fse::g_timing.on = on != 0;
    return FSE_OK;
}

int fse_timing_read(double *ms, int64_t *window_launches, int64_t *calls) {
    double tot = 0.0;
    const long long n = (long long)fse::g_timing.ev.size();
    for (auto &e : fse::g_timing.ev) {
        float t = 0.f;
        cudaError_t ce = cudaEventSynchronize(e.second);
        if (ce == cudaSuccess) ce = cudaEventElapsedTime(&t, e.first, e.second);
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
        if (ce != cudaSuccess) {
            fse::g_timing.ev.clear();
            return fail(FSE_ECUDA, std::string("timing: ") + cudaGetErrorString(ce));
        }
        tot += t;
    }
    fse::g_timing.ev.clear();
    cudaDeviceSynchronize();
    for (auto &r : fse::g_timing.redo) {
        for (int i = 0; i < r.second; ++i) fse::g_redo_total += r.first[i];
        cudaFreeHost(r.first);
    }
    fse::g_timing.redo.clear();
    if (ms) *ms = tot;
    if (window_launches) *window_launches = fse::g_timing.window_launches;
    if (calls) *calls = n;
    fse::g_timing.window_launches = 0;
    return FSE_OK;
}

int fse_fma_probe(int32_t kind, int32_t blocks, int32_t threads, int32_t iters, void *scratch,
                  void *stream) {
    if (blocks < 1 || threads < 32 || iters < 1 || !scratch) return fail(FSE_EINVAL, "bad probe shape");
    cudaStream_t st = (cudaStream_t)stream;
    if (kind == 0)
        fse::fma_probe_kernel<<<blocks, threads, 0, st>>>((float *)scratch, iters, 0.999999f, 1e-7f);
    else if (kind == 1)
        fse::fma2_probe_kernel<<<blocks, threads, 0, st>>>((float *)scratch, iters, 0.999999f, 1e-7f);
    else if (kind == 2)
        fse::dfma_probe_kernel<<<blocks, threads, 0, st>>>((float *)scratch, iters, 0.999999, 1e-7);
    else
        return fail(FSE_EINVAL, "probe kind");
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return fail(FSE_ECUDA, cudaGetErrorString(ce));
    return FSE_OK;
}

int fse_set_guard(double tau0, double tau1) {
    fse::g_tau0 = tau0;
    fse::g_tau1 = tau1;
    return FSE_OK;
}

int fse_set_dataflow(int32_t on) {
    fse::g_dataflow = on != 0;
    return FSE_OK;
}

int64_t fse_guard_redo_count(int32_t reset) {
    const long long v = fse::g_redo_total;
    if (reset) fse::g_redo_total = 0;
    return v;
}

int64_t fse_launch_count(int32_t reset) {
    return reset ? fse::g_launches.exchange(0) : fse::g_launches.load();
}

int fse_run_windows(int32_t n, int32_t M, int32_t N, int32_t F1, int32_t F2, const void *values,
                    const void *weights, int32_t iterations, double gamma, int32_t dtype,
                    int32_t *picks, void *plog, void *energies, void *residual, void *stream) {
    if (n < 0 || M < 1 || N < 1 || F1 < M || F2 < N || iterations < 0)
        return fail(FSE_EINVAL, "bad window / DFT shape");
    if (F1 > 0xFFFF / F2) return fail(FSE_EINVAL, "DFT too large");
    if (!(gamma > 0.0 && gamma <= 1.0)) return fail(FSE_EINVAL, "gamma must lie in (0, 1]");
    if (!values || !weights || ((!picks || !plog) && iterations > 0))
        return fail(FSE_EINVAL, "NULL buffer");
    if ((energies == nullptr) != (residual == nullptr))
        return fail(FSE_EINVAL, "energies and residual go together");
    if (dtype != FSE_F64 && dtype != FSE_F32) return fail(FSE_EINVAL, "dtype");
    fse::KArgs a{};
    a.values = values;
    a.weights = weights;
    a.plog = plog;
    a.energies = energies;
    a.residual = residual;
    a.M = M;
    a.N = N;
    a.F1 = F1;
    a.F2 = F2;
    a.iterations = iterations;
    a.gamma = gamma;
    a.picks = picks;
    cudaStream_t s = (cudaStream_t)stream;
    const bool dbg = energies != nullptr;
    if (!dbg && F1 == F2 && fse::fast_supported(dtype, F1, M, N, 0)) {
        fse::FastArgs f{};
        f.values = values;
        f.weights = weights;
        f.plog = plog;
        f.M = M;
        f.N = N;
        f.iterations = iterations;
        f.gamma = gamma;
        f.picks = picks;
        return fse::fast_windows(dtype, F1, f, n, s);
    }
    if (dtype == FSE_F64)
        return dbg ? fse::dispatch<double, 1, true>(a, n, M, N, F1, F2, 0, s)
                   : fse::dispatch<double, 1, false>(a, n, M, N, F1, F2, 0, s);
    return dbg ? fse::dispatch<float, 1, true>(a, n, M, N, F1, F2, 0, s)
               : fse::dispatch<float, 1, false>(a, n, M, N, F1, F2, 0, s);
}

int fse_conceal_frames(int32_t n, FsePlan *const *plans, void *const *images,
                       const uint8_t *const *masks, uint8_t *const *masks_out,
                       const FseParamsC *p, int32_t dtype, const void *decay, int32_t decay_dim,
                       int32_t *picks, void *stream) {
    if (n < 0 || (n > 0 && (!plans || !images || !masks || !p || !decay)))
        return fail(FSE_EINVAL, "NULL argument");
    if (n == 0) return FSE_OK;
    if (dtype != FSE_F64 && dtype != FSE_F32) return fail(FSE_EINVAL, "dtype");
    const fse::Plan &P0 = plans[0]->p;
    for (int f = 0; f < n; ++f) {
        const fse::Plan &P = plans[f]->p;
        if (!images[f] || !masks[f]) return fail(FSE_EINVAL, "NULL image/mask");
        if (P.H != P0.H || P.W != P0.W || P.B != P0.B || P.d != P0.d)
            return fail(FSE_EINVAL, "plans of one call must share image size, block size and d");
    }
    if (P0.B != p->block_size || P0.d != p->d || P0.iterations != p->iterations)
        return fail(FSE_EINVAL, "params do not match the plan");
    const int F1 = p->fft1, F2 = p->fft2;
    if ((F1 == 0) != (F2 == 0)) return fail(FSE_EINVAL, "fft1/fft2 must both be 0 or both set");
    if (F1 && (F1 < P0.max_wr || F2 < P0.max_wc))
        return fail(FSE_EINVAL, "FFT size smaller than the largest window");
    if (F1 && F1 > 0xFFFF / F2) return fail(FSE_EINVAL, "DFT too large");
    if (decay_dim < std::max(P0.max_wr, P0.max_wc)) return fail(FSE_EINVAL, "decay table too small");

    const int nb = P0.rows * P0.cols;
    int n_levels = 0;
    for (int f = 0; f < n; ++f) n_levels = std::max(n_levels, (int)plans[f]->p.level_ptr.size() - 1);
    // merged level lists: level L of every frame in one launch
    std::vector<int> lvl_off(n_levels + 1, 0);
    size_t n_entries = 0;
    for (int l = 0; l < n_levels; ++l) {
        lvl_off[l] = (int)n_entries;
        for (int f = 0; f < n; ++f) {
            const fse::Plan &P = plans[f]->p;
            if (l + 1 < (int)P.level_ptr.size()) n_entries += P.level_ptr[l + 1] - P.level_ptr[l];
        }
    }
    lvl_off[n_levels] = (int)n_entries;
    // one device staging buffer:
    //   uploaded: frame table | ranks | entries (level order)
    //   zeroed:   redo counters | work counter | completion flags
    //   scratch:  redo list
    auto up256 = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t off_rank = up256(sizeof(fse::FrameDesc) * n);
    const size_t off_ent = off_rank + up256(sizeof(int32_t) * (size_t)nb * n);
    const size_t off_cnt = off_ent + up256(sizeof(int2) * std::max<size_t>(n_entries, 1));
    const size_t off_next = off_cnt + up256(sizeof(int) * std::max(n_levels, 1));
    const size_t off_done = off_next + 256;
    const size_t off_queue = off_done + up256(sizeof(int) * (size_t)nb * n);
    const size_t off_redo = off_queue + up256(sizeof(int) * std::max<size_t>(n_entries, 1));
    const size_t bytes = off_redo + sizeof(int2) * std::max<size_t>(n_entries, 1);
    std::vector<unsigned char> host(off_cnt);
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *dev = nullptr;
    FSE_CUDA_TRY(cudaMallocAsync((void **)&dev, bytes, s));
    fse::FrameDesc *fdh = reinterpret_cast<fse::FrameDesc *>(host.data());
    int32_t *rk = reinterpret_cast<int32_t *>(host.data() + off_rank);
    int2 *ent = reinterpret_cast<int2 *>(host.data() + off_ent);
    for (int f = 0; f < n; ++f) {
        fdh[f].image = images[f];
        fdh[f].mask = masks[f];
        fdh[f].mask_out = masks_out ? masks_out[f] : nullptr;
        fdh[f].rank = reinterpret_cast<const int32_t *>(dev + off_rank) + (size_t)f * nb;
        std::memcpy(rk + (size_t)f * nb, plans[f]->p.rank.data(), sizeof(int32_t) * nb);
    }
    {
        size_t k = 0;
        for (int l = 0; l < n_levels; ++l)
            for (int f = 0; f < n; ++f) {
                const fse::Plan &P = plans[f]->p;
                if (l + 1 >= (int)P.level_ptr.size()) continue;
                for (int i = P.level_ptr[l]; i < P.level_ptr[l + 1]; ++i) ent[k++] = make_int2(f, P.level_blocks[i]);
            }
    }
    // pageable source: staged by the driver before returning, so `host` may go
    cudaError_t ce = cudaMemcpyAsync(dev, host.data(), off_cnt, cudaMemcpyHostToDevice, s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(dev + off_cnt, 0, off_queue - off_cnt, s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(dev + off_queue, 0xFF, off_redo - off_queue, s);
    if (ce != cudaSuccess) {
        cudaFreeAsync(dev, s);
        return fail(FSE_ECUDA, std::string("upload: ") + cudaGetErrorString(ce));
    }
    fse::KArgs a{};
    a.frames = reinterpret_cast<const fse::FrameDesc *>(dev);
    a.H = P0.H;
    a.W = P0.W;
    a.B = P0.B;
    a.d = P0.d;
    a.rows = P0.rows;
    a.cols = P0.cols;
    a.delta = p->delta;
    a.decay = reinterpret_cast<const double *>(decay);
    a.decay_dim = decay_dim;
    a.F1 = F1;
    a.F2 = F2;
    a.iterations = p->iterations;
    a.gamma = p->gamma;
    a.picks = picks;
    const int Mmax = P0.max_wr, Nmax = P0.max_wc, model_n = P0.B * P0.B;
    int rc = FSE_OK;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (fse::g_timing.on) {
        if (cudaEventCreate(&ev0) != cudaSuccess || cudaEventCreate(&ev1) != cudaSuccess) {
            cudaFreeAsync(dev, s);
            return fail(FSE_ECUDA, "event create");
        }
        cudaEventRecord(ev0, s);
    }
    const bool fast = F1 == F2 && fse::fast_supported(dtype, F1, Mmax, Nmax, model_n);
    int n_levels_run = n_levels;
    const bool guard = fast && dtype == FSE_F32 && fse::g_tau0 >= 0.0 && F1 != 128;
    fse::FastArgs f{};
    if (fast) {
        f.frames = a.frames;
        f.H = a.H;
        f.W = a.W;
        f.B = a.B;
        f.d = a.d;
        f.rows = a.rows;
        f.cols = a.cols;
        f.delta = a.delta;
        f.decay = a.decay;
        f.decay_dim = a.decay_dim;
        f.iterations = a.iterations;
        f.gamma = a.gamma;
        f.picks = a.picks;
        f.tau0 = (float)fse::g_tau0;
        f.tau1 = (float)fse::g_tau1;
    }
    int2 *redo = reinterpret_cast<int2 *>(dev + off_redo);
    int *counters = reinterpret_cast<int *>(dev + off_cnt);
    if (fast && !guard && fse::dataflow_enabled()) {
        // one persistent launch over all levels of all frames (fse_fast.cuh)
        f.entries = reinterpret_cast<const int2 *>(dev + off_ent);
        f.total = (int)n_entries;
        f.next = reinterpret_cast<int *>(dev + off_next);
        f.done = reinterpret_cast<int *>(dev + off_done);
        f.queue = reinterpret_cast<int *>(dev + off_queue);
        f.R = (P0.d + P0.B - 1) / P0.B;
        if (n_entries > 0) rc = fse::fast_dataflow(dtype, F1, f, Mmax, Nmax, model_n, s);
        if (fse::g_timing.on) ++fse::g_timing.window_launches;
        n_levels_run = 0;
    }
    for (int l = 0; l < n_levels_run && rc == FSE_OK; ++l) {
        const int2 *lvl = reinterpret_cast<const int2 *>(dev + off_ent) + lvl_off[l];
        const int cnt = lvl_off[l + 1] - lvl_off[l];
        if (cnt == 0) continue;
        if (fast) {
            f.entries = lvl;
            f.redo_list = redo + lvl_off[l];
            f.redo_count = counters + l;
            rc = fse::fast_level(dtype, F1, guard, f, cnt, Mmax, Nmax, model_n, s);
            if (rc == FSE_OK && guard) {
                fse::FastArgs r = f;
                r.entries = redo + lvl_off[l];
                r.count = counters + l;
                rc = fse::fast_redo(F1, r, cnt, Mmax, Nmax, model_n, s);
            }
        } else {
            a.entries = lvl;
            rc = dtype == FSE_F64 ? fse::dispatch<double, 0, false>(a, cnt, Mmax, Nmax, F1, F2, model_n, s)
                                  : fse::dispatch<float, 0, false>(a, cnt, Mmax, Nmax, F1, F2, model_n, s);
        }
        if (fse::g_timing.on) ++fse::g_timing.window_launches;
    }
    if (fse::g_timing.on && guard && n_levels > 0) {
        int *hc = nullptr;
        if (cudaMallocHost((void **)&hc, sizeof(int) * n_levels) == cudaSuccess) {
            cudaMemcpyAsync(hc, counters, sizeof(int) * n_levels, cudaMemcpyDeviceToHost, s);
            fse::g_timing.redo.emplace_back(hc, n_levels);
        }
    }
    if (fse::g_timing.on) {
        cudaEventRecord(ev1, s);
        fse::g_timing.ev.emplace_back(ev0, ev1);
    }
    if (rc == FSE_OK && masks_out) {
        const long long total = (long long)n * P0.H * P0.W;
        int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
        fse::finalize_masks_kernel<<<grid, 256, 0, s>>>(a.frames, n, P0.H, P0.W, P0.B, P0.cols);
        ce = cudaGetLastError();
        if (ce != cudaSuccess) rc = fail(FSE_ECUDA, std::string("finalize: ") + cudaGetErrorString(ce));
        else fse::g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    cudaFreeAsync(dev, s);
    return rc;
}

}  // extern "C"
