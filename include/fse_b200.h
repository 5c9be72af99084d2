/*
 * fse_b200.h — C ABI of the B200-native Frequency Selective Extrapolation (FSE)
 * hot path.  Built into paper_2207_00233_b200/libfse_b200.so (sm_100a).
 *
 * Plain C types only (no torch types).  Device pointers are CUDA device
 * addresses; `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 * Every function returns FSE_OK (0) or a negative errno-style code; the message
 * of the last failure on the calling thread is available from fse_last_error().
 * No C++ exception crosses this boundary.  Functions are re-entrant; memory
 * passed in is caller-owned.
 *
 * Each entry point names the reference interface it replaces
 * (reference = /root/reference/pkg/src/fsefill, the `fsefill` package).
 */
#ifndef FSE_B200_H
#define FSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSE_OK 0
#define FSE_EINVAL (-22)   /* bad argument (mirrors the reference's ValueError) */
#define FSE_ENOMEM (-12)
#define FSE_ECUDA (-5)     /* CUDA runtime error */
#define FSE_ENOTSUP (-95)  /* configuration not compiled in (e.g. FFT size) */

/* arithmetic type of the device path */
#define FSE_F64 0
#define FSE_F32 1

/* processing orders, fsefill.conceal.LINESCAN / OPTIMIZED (conceal.py:30-32) */
#define FSE_ORDER_OPTIMIZED 0
#define FSE_ORDER_LINESCAN 1

/* sample states of a loss mask, fsefill.image KNOWN/LOST/RECONSTRUCTED (image.py:14-16) */
#define FSE_KNOWN 0
#define FSE_LOST 1
#define FSE_RECONSTRUCTED 2

/* fsefill.fse.FseParams (fse.py:55-86) plus the DFT size.
 * fft1 = fft2 = 0 keeps the reference semantics (DFT size = window shape,
 * fse.py:158-159); otherwise every window is zero-padded at the top-left to
 * fft1 x fft2, which must be >= the largest window. */
typedef struct FseParamsC {
    int32_t d;           /* border width in samples */
    int32_t block_size;  /* B: side of the square block grid */
    int32_t iterations;  /* basis-selection iterations */
    int32_t fft1, fft2;  /* DFT size, 0 = window shape */
    double rho;          /* isotropic decay in (0, 1) */
    double delta;        /* reconstructed-sample down-weighting in [0, 1] */
    double gamma;        /* ODC damping in (0, 1] */
} FseParamsC;

const char *fse_last_error(void);

/* Library/device self-description: writes up to n ints:
 * [abi_version, n_fast_fft_sizes, fast sizes..., sm_count(or -1 w/o device)] */
int fse_version(int32_t *out, int32_t n);

/* ------------------------------------------------------------------------
 * Per-window operator.
 * Replaces fsefill._kernel.run_fse(values, weights, iterations, gamma)
 * (_kernel.pyx:128-187, contract _kernel_py.py:13-30), called once per window
 * by fsefill.fse.generate_model (fse.py:153-156).  Batched: n windows of
 * M x N samples, each zero-padded at the top-left to an F1 x F2 DFT.
 *   values, weights : device, dtype, [n][M][N] row-major; weights >= 0 and
 *                     positive somewhere (the reference's precondition, enforced
 *                     upstream by DegenerateWindowError, fse.py:150-151)
 *   picks           : device int32 [n][iterations][2]   (required)
 *   plog            : device dtype [n][iterations][2]   (required) projection
 *                     coefficient p = g[a,b] / sum(w) of every pick; the host
 *                     replays coeff[a,b] += gamma*p exactly as _kernel.pyx:50-71
 *   energies        : device dtype [n][iterations+1] or NULL (debug)
 *   residual        : device dtype [n][M][N] or NULL (debug, weighted residual r)
 * energies and residual must be both NULL or both non-NULL.  The synthesis
 * (fse.py:159) is the host's ifft2 of the replayed coefficient grid. */
int fse_run_windows(int32_t n, int32_t M, int32_t N, int32_t F1, int32_t F2,
                    const void *values, const void *weights,
                    int32_t iterations, double gamma, int32_t dtype,
                    int32_t *picks, void *plog, void *energies, void *residual,
                    void *stream);

/* ------------------------------------------------------------------------
 * Scheduler + plan (host C++).
 * Replaces the order logic of fsefill.conceal.conceal (conceal.py:97-181):
 * grid (grid.py:81-144), neighbour-count wavefront scheduler
 * (schedule.py:28-105), snapshot semantics (conceal.py:148-163), deferral of
 * degenerate windows and retry sweeps (conceal.py:69-94).  The plan assigns
 * every lossy block an effective rank (its phase; retries after all phases),
 * decides degeneracy on the host (pure function of mask and ranks), and groups
 * blocks into dependency levels: a block depends only on lower-rank blocks
 * whose samples its window covers, so one level = one batched launch. */
typedef struct FsePlan FsePlan;

int fse_plan_build(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p,
                   int32_t order, FsePlan **out);
/* fse_plan_build on n_threads host threads (0 = automatic: FSE_PLAN_THREADS or
 * 3/4 of the usable CPUs for grids of >= 65536 blocks; 1 = the sequential planner).
 * The optimized order is planned by bands of block rows, one per thread, with
 * a per-phase minimum, a first-row fix-up and band-local commits; the plan is
 * identical for every thread count. */
int fse_plan_build_threads(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p,
                           int32_t order, int32_t n_threads, FsePlan **out);
/* n masks (each H x W) built on n_threads host threads (0 = hardware) */
int fse_plan_build_many(int32_t n, const uint8_t *const *masks, int32_t H, int32_t W,
                        const FseParamsC *p, int32_t order, int32_t n_threads,
                        FsePlan **out);
void fse_plan_free(FsePlan *plan);

/* sizes[0..9] = rows, cols, n_lossy, n_processed, n_batches, n_batch_entries,
 *               n_levels, n_unconcealed, max_window_rows, max_window_cols */
int fse_plan_sizes(const FsePlan *plan, int32_t *sizes);
/* ConcealReport.batches (conceal.py:35-42): CSR, ptr[n_batches+1] */
int fse_plan_batches(const FsePlan *plan, int32_t *ptr, int32_t *blocks);
/* dependency levels, CSR over processed blocks, ptr[n_levels+1] */
int fse_plan_levels(const FsePlan *plan, int32_t *ptr, int32_t *blocks);
/* Level balancing of a built plan (no reference counterpart: the reference's
 * batches, conceal.py:148-163, stay as they are; this only changes in which
 * LAUNCH a block runs).  Every block sits at its earliest dependency level;
 * blocks with slack (no dependent needs them yet) move from levels wider than
 * max(narrow, wave) windows into later levels that still have free slots: up
 * to `narrow` windows in levels that stay at most that wide (the caller passes
 * the SM count: those levels run one window per SM), and, if wave > 0, up to
 * `wave` in levels of at most `wave` windows (the resident windows of one wave).
 * Ranks, batches and results are unchanged (only true dependences order the
 * launches).  narrow = 0 leaves the plan as it is.  *moved (optional) = blocks
 * that changed level. */
int fse_plan_rebalance(FsePlan *plan, int32_t narrow, int32_t wave, int32_t *moved);
/* effective rank per block (INT32_MAX = not processed) [rows*cols] */
int fse_plan_ranks(const FsePlan *plan, int32_t *rank);
/* ConcealReport.unconcealed_blocks, row-major */
int fse_plan_unconcealed(const FsePlan *plan, int32_t *blocks);
/* A plan as bytes (ranks, batch and level CSRs, unconcealed list, geometry and
 * parameters): one rank plans a large frame and broadcasts them, the other
 * ranks import instead of re-planning (strips.py).  export_size < 0 = error. */
int64_t fse_plan_export_size(const FsePlan *plan);
int fse_plan_export(const FsePlan *plan, void *buf, int64_t size);
int fse_plan_import(const void *buf, int64_t size, FsePlan **out);

/* fsefill.schedule.init_counts (schedule.py:28-57): lossy[rows*cols] != 0 marks
 * a lossy block; counts[rows*cols] out. */
int fse_init_counts(const uint8_t *lossy, int32_t rows, int32_t cols, int32_t *counts);
/* fsefill.schedule.schedule_all (schedule.py:97-105): batches as CSR.
 * ptr needs room for (#pending + 1) entries, blocks for #pending. */
int fse_schedule_all(const int32_t *counts, int32_t rows, int32_t cols,
                     int32_t *ptr, int32_t *blocks, int32_t *n_batches);

/* ------------------------------------------------------------------------
 * Device pipeline.
 * Replaces the per-batch loop of fsefill.conceal.conceal (conceal.py:145-163:
 * classify_window + _snapshot + extrapolate_block + _write_block) for n frames
 * that share H, W and params.  Level by level (levels of all frames merged into
 * one launch), one CTA per block: area classification from the original mask
 * and the plan's ranks (grid.py:108-135), weights (fse.py:105-119), DFT set-up,
 * the iterative model fit, and write-back of the block's LOST samples
 * (conceal.py:61-66).
 *   images    : n device pointers, dtype, [H][W], updated in place
 *   masks     : n device pointers, uint8 [H][W], the ORIGINAL masks (read only)
 *   masks_out : n device pointers, uint8 [H][W] or NULL: LOST samples of
 *               concealed blocks become RECONSTRUCTED (may alias masks only if
 *               the caller no longer needs the original)
 *   decay     : device dtype table, decay[i*decay_dim + j] = rho ** sqrt((i/2)^2 + (j/2)^2)
 *               for i, j = |2*offset| from the window centre (fse.py:112-115)
 *   picks     : device int32 [n][rows*cols][iterations][2] or NULL (parity/debug) */
int fse_conceal_frames(int32_t n, FsePlan *const *plans, void *const *images,
                       const uint8_t *const *masks, uint8_t *const *masks_out,
                       const FseParamsC *p, int32_t dtype,
                       const void *decay, int32_t decay_dim,
                       int32_t *picks, void *stream);

/* fp32 near-tie guard of the fast path (F = 32/64): a window whose runner-up
 * energy comes within (tau0 + tau1 * iteration) of the maximum is recomputed
 * by the fp64 kernel before the next level.  tau0 < 0 disables the guard.
 * Default: off (tau0 = -1).  Process-wide. */
int fse_set_guard(double tau0, double tau1);
/* fse_conceal_frames execution mode for the fast path: 1 = one persistent
 * dataflow launch (ready queue over per-block dependency counters; blocks start
 * when their own inputs are written), 0 (default) = one launch per dependency
 * level.  Results are identical.  Process-wide; FSE_DATAFLOW=1 sets the default. */
int fse_set_dataflow(int32_t on);
/* Frame groups of one fse_conceal_frames call (level-launch mode): the frames
 * are split into n contiguous groups of about equal work whose level sequences
 * run on forked streams, so one group's partial last wave of a level overlaps
 * another group's work.  1..8, default 2 (FSE_GROUPS sets the default).
 * Results are identical for every n.  Process-wide. */
int fse_set_groups(int32_t n);
/* Weight-spectrum cache of a session (fast path): W = fft2(w) of
 * _kernel.pyx:148 depends only on a window's shape and class map
 * (fse.py:105-119), so windows of one call that share both share W.  1
 * (default; FSE_WCACHE=0 sets the default off): before the first level every
 * window's class map is hashed and compared on the device (F >= 64; sessions
 * of >= 2,048 windows and >= 1,024 windows per level on average: a plane per
 * map shared by >= 2 windows; sessions of narrower levels and >= 1,024 windows:
 * a plane for every window, if the plane capacity covers them), each W shared by
 * >= 2 windows is computed once, and the level kernels load it instead of
 * running the weight half of their set-up.  Results are bit-identical to 0
 * (every window computes its own W).  Process-wide. */
int fse_set_wcache(int32_t on);
/* Totals over the sessions read back by fse_timing_read so far: windows
 * classified, windows that loaded a cached W, planes wanted (distinct shared
 * maps; may exceed the plane capacity).  reset != 0 clears them. */
int fse_wcache_stats(int64_t *windows, int64_t *hits, int64_t *planes, int32_t reset);
/* fp32 argmax form per level launch: launches of fewer windows than this use
 * the tracked argmax (each thread carries its best bin; one barrier per
 * iteration), wider ones the lazy argmax (running maximum only; the winning
 * warp re-finds its bin after a second barrier).  Same argmax, identical
 * results; tracked is faster on narrow (latency-bound) levels.  Default
 * 16 x SM count (FSE_TRACK_BELOW sets the default); 0 = always lazy.
 * Process-wide. */
int fse_set_track_below(int32_t windows);
/* Windows redone in fp64 by the guard, summed over timed calls (fse_timing_*). */
int64_t fse_guard_redo_count(int32_t reset);

/* ------------------------------------------------------------------------
 * Row-band shards of one frame (spatial strip sharding across GPUs, BASELINE
 * config 5).  Every rank builds the same global plan
 * (fse_plan_build is deterministic), opens a shard over its band of block rows
 * [row_lo, row_hi) on its own device copy of the frame, and then alternates
 * fse_shard_run over one level with a halo exchange: the image rows of the
 * R = ceil(d/B) block rows at each band edge go to the neighbouring rank
 * whenever that level wrote blocks there (edge_flags bit 0 = top zone,
 * bit 1 = bottom zone).  Masks and ranks never change, so only image samples
 * cross devices.  Same semantics as fse_conceal_frames on the whole frame.
 * Replaces the batch loop of conceal() (conceal.py:145-163) for one band. */
typedef struct FseShard FseShard;
int fse_shard_open(const FsePlan *plan, int32_t row_lo, int32_t row_hi, void *image,
                   const uint8_t *mask, uint8_t *mask_out, const FseParamsC *p, int32_t dtype,
                   const void *decay, int32_t decay_dim, void *stream, FseShard **out);
/* number of levels and, if edge_flags != NULL, int32[n_levels] edge flags */
int fse_shard_levels(const FseShard *shard, int32_t *n_levels, int32_t *edge_flags);
/* launch levels [level_lo, level_hi) of the band's blocks on stream */
int fse_shard_run(FseShard *shard, int32_t level_lo, int32_t level_hi, void *stream);
/* mask pass over the band's rows (if mask_out was given) and release */
int fse_shard_close(FseShard *shard, void *stream);

/* Fused halo exchange over peer memory (NVLink / NVSwitch), replacing the
 * per-level NCCL send/recv of the protocol above: the level kernel's
 * write-back also stores the band-edge blocks (block rows within R of the
 * edge) straight into the neighbour's frame, and per level the shard signals
 * the neighbours through device flags; before level l its stream waits (a
 * front-end cuStreamWaitValue32, no spinning SM) until both neighbours have
 * completed level l-1, and after the last level until they are done writing
 * into this frame.  The whole level sequence is then one fse_shard_run call
 * with no host round trips.  Peer frames and flags are CUDA IPC mappings
 * (one process per GPU).  Same results as the NCCL protocol.
 * Handles are FSE_IPC_HANDLE_BYTES opaque bytes (allocation handle + offset). */
#define FSE_IPC_HANDLE_BYTES 72
int fse_ipc_handle(const void *dev_ptr, void *handle);
int fse_ipc_open(const void *handle, void **dev_ptr);
int fse_ipc_close(void *dev_ptr);
/* two zeroed uint32 device flags: [0] from the upper neighbour, [1] from the lower */
int fse_flags_alloc(uint32_t **flags);
int fse_flags_free(uint32_t *flags);
/* neighbours' frames and flags (NULL = no neighbour on that side), this
 * rank's own flags, and the run's flag base (identical on every rank).  The
 * run's flag values lie in [base, base + n_levels]; a caller reusing the
 * flags passes, for each run, a base above the previous run's last value
 * (base_next = base + n_levels + 1; flags start at 0, so the first base is
 * >= 1), so values of one run never satisfy another's waits whatever the
 * runs' level counts.  A run starting at level 0 first signals "frame
 * initialised" and waits for the neighbours' signal, so work queued before it
 * on the stream (a frame reset) precedes every peer store into this frame.
 * All-NULL peers detach the shard (always allowed).  FSE_ENOTSUP when the
 * shard cannot fuse the exchange (not the fast kernel, or several frames):
 * callers then agree on the collective exchange (strips.conceal_strips). */
int fse_shard_set_peers(FseShard *shard, void *up_image, uint32_t *up_flags, void *down_image,
                        uint32_t *down_flags, uint32_t *own_flags, uint32_t base);

/* Output epilogue over n frames of npix samples each (device pointers, frames
 * contiguous): out_u8 (or NULL) = floor(clip(x, 0, 255) + 0.5), the rounding
 * of fsefill.image.save_pgm (image.py:79-88); if sums != NULL, per frame f
 * sums[2f] = sum (truth - x)^2 and sums[2f+1] = count over samples whose mask
 * is not KNOWN — the terms of fsefill.evalkit.psnr (evalkit.py:67-81).
 * truth: uint8 originals; masks: uint8 (pre- or post-concealment). */
int fse_quantize_psnr(int32_t n, int64_t npix, const void *images, int32_t dtype, const uint8_t *truth,
                      const uint8_t *masks, uint8_t *out_u8, double *sums, void *stream);

/* Count of kernel launches issued since the last reset (bench.py gpu_launches). */
int64_t fse_launch_count(int32_t reset);

/* Device timing of the window-kernel launches of fse_conceal_frames on the
 * calling thread: enable, run, then read the summed CUDA-event time of the
 * level launches (ms), how many window-kernel launches that covered and how
 * many calls; reading resets.  Used by bench.py for the roofline. */
int fse_timing_enable(int32_t on);
int fse_timing_read(double *ms, int64_t *window_launches, int64_t *calls);

/* Arithmetic throughput probes (roofline denominators): blocks x threads
 * threads, each running 8 independent FMA chains for iters steps.
 * kind 0: FFMA (16*iters FLOP per thread), 1: FFMA2 / packed f32x2
 * (32*iters), 2: DFMA (16*iters).  scratch: device float[1]. */
int fse_fma_probe(int32_t kind, int32_t blocks, int32_t threads, int32_t iters, void *scratch,
                  void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FSE_B200_H */
