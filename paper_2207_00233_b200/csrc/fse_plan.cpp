// Host scheduler for the FSE hot path (C++, no CUDA).
//
// Reference behaviour being reproduced (reference = /root/reference/pkg/src/fsefill):
//   block grid, ragged edges            grid.py:26-88
//   per-block lost tally                grid.py:138-144
//   neighbour counts + rim bonus        schedule.py:28-57
//   N_min batch selection, commit       schedule.py:60-105  (Algorithm 1)
//   snapshot-then-write batches         conceal.py:145-163
//   linescan order                      conceal.py:133-143
//   deferral + retry sweeps             conceal.py:54-58, 69-94
//
// The device never replays the reference's mutable mask.  Instead every lossy
// block gets an effective rank (the index of the reference batch that writes
// it; retries follow all batches), and a lost sample s seen from block b is
// "reconstructed" (area R) iff the block owning s has a smaller rank than b.
// That is a pure function of (original mask, ranks), so blocks of different
// reference batches may share a launch as long as every lower-rank block whose
// samples their window covers has finished: those dependencies define levels.
#include <algorithm>
#include <functional>
#include <atomic>
#include <climits>
#include <limits>
#include <cstring>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#ifdef __linux__
#include <sched.h>
#endif

#include "fse_common.h"

namespace fse {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

namespace {

constexpr int kMarginBonus = 3;  // schedule.py:20
constexpr int kCornerBonus = 5;  // schedule.py:21

int validate(const FseParamsC *p, int32_t H, int32_t W, int32_t order) {
    if (!p) return fail(FSE_EINVAL, "params is NULL");
    if (H < 1 || W < 1) return fail(FSE_EINVAL, "image dimensions must be positive");
    if (p->d < 0) return fail(FSE_EINVAL, "d must be >= 0");
    if (!(p->rho > 0.0 && p->rho < 1.0)) return fail(FSE_EINVAL, "rho must lie in (0, 1)");
    if (!(p->delta >= 0.0 && p->delta <= 1.0)) return fail(FSE_EINVAL, "delta must lie in [0, 1]");
    if (!(p->gamma > 0.0 && p->gamma <= 1.0)) return fail(FSE_EINVAL, "gamma must lie in (0, 1]");
    if (p->iterations < 0) return fail(FSE_EINVAL, "iterations must be >= 0");
    if (p->block_size < 1) return fail(FSE_EINVAL, "block_size must be >= 1");
    if (order != FSE_ORDER_OPTIMIZED && order != FSE_ORDER_LINESCAN)
        return fail(FSE_EINVAL, "unknown order");
    return FSE_OK;
}

// schedule.py:28-57 on a row-major lossy table
void init_counts_impl(const uint8_t *lossy, int rows, int cols, int32_t *counts) {
    // 3x3 box sums of the lossy map through a zero-padded copy (no bounds
    // tests in the inner loop), minus the block itself
    const int pc = cols + 2;
    std::vector<uint8_t> pad((size_t)(rows + 2) * pc, 0);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) pad[(size_t)(r + 1) * pc + c + 1] = lossy[(size_t)r * cols + c] ? 1 : 0;
    std::vector<uint8_t> h3((size_t)(rows + 2) * cols);  // horizontal 3-sums of each padded row
    for (int r = 0; r < rows + 2; ++r) {
        const uint8_t *p = &pad[(size_t)r * pc];
        uint8_t *o = &h3[(size_t)r * cols];
        for (int c = 0; c < cols; ++c) o[c] = (uint8_t)(p[c] + p[c + 1] + p[c + 2]);
    }
    for (int r = 0; r < rows; ++r) {
        const uint8_t *a = &h3[(size_t)r * cols], *m = &h3[(size_t)(r + 1) * cols], *z = &h3[(size_t)(r + 2) * cols];
        const int er = (r == 0) + (r == rows - 1);
        for (int c = 0; c < cols; ++c) {
            const int self = lossy[(size_t)r * cols + c] ? 1 : 0;
            int n = a[c] + m[c] + z[c] - self;
            const int edges = er + (c == 0) + (c == cols - 1);
            if (edges == 1) n += kMarginBonus;
            else if (edges >= 2) n += kCornerBonus;
            counts[(size_t)r * cols + c] = self ? n : -1;
        }
    }
}

// Largest pending count schedule_impl accepts (one bucket per value); the
// reference's init_counts produces at most 8 + 5.
constexpr int kMaxCount = 1 << 14;

// schedule.py:60-105 with a bucket queue: one bitset of pending blocks per
// count value, scanned in row-major order for the current minimum.  Selection
// of a whole batch happens before any commit, as in select_batch/commit_batch.

template <typename CT>
void schedule_loop(const int32_t *counts_in, int rows, int cols, int maxc, long pending,
                   std::vector<int32_t> &ptr, std::vector<int32_t> &blocks);

int schedule_impl(const int32_t *counts_in, int rows, int cols,
                  std::vector<int32_t> &ptr, std::vector<int32_t> &blocks) {
    const int nb = rows * cols;
    // Pending counts (>= 0) fit in int8 for init_counts' counts (<= 13) and in
    // int16 up to kMaxCount; everything below 0 is done and its exact value
    // never matters again (select_batch only looks at counts >= 0,
    // schedule.py:69-70), so done blocks are kept at -1 instead of drifting.
    int maxc = 0;
    long pending = 0;
    for (int b = 0; b < nb; ++b)
        if (counts_in[b] >= 0) {
            if (counts_in[b] > kMaxCount)
                return fail(FSE_EINVAL, "count " + std::to_string(counts_in[b]) + " above the supported " +
                                            std::to_string(kMaxCount));
            maxc = std::max(maxc, (int)counts_in[b]);
            ++pending;
        }
    if (maxc <= 126) schedule_loop<int8_t>(counts_in, rows, cols, maxc, pending, ptr, blocks);
    else schedule_loop<int16_t>(counts_in, rows, cols, maxc, pending, ptr, blocks);
    return FSE_OK;
}

template <typename CT>
void schedule_loop(const int32_t *counts_in, int rows, int cols, int maxc, long pending,
                   std::vector<int32_t> &ptr, std::vector<int32_t> &blocks) {
    const int nb = rows * cols;
    const int words = (nb + 63) / 64;
    std::vector<CT> cnt(nb);
    for (int b = 0; b < nb; ++b) cnt[b] = (CT)(counts_in[b] >= 0 ? counts_in[b] : -1);
    // bucket c: bitset of pending blocks with count c; summary: bitset of its
    // non-zero words, so a row-major scan skips empty stretches 64 words at a
    // time.  The count is the fast index of both arrays: a neighbour's move
    // from bucket c to c - 1 touches one cache line, not two far-apart ones.
    const int NC = maxc + 1;
    const int swords = (words + 63) / 64;
    std::vector<uint64_t> bits((size_t)words * NC, 0), summ((size_t)swords * NC, 0);
    std::vector<long> bsize(NC, 0);
    auto add = [&](int c, int b) {
        bits[(size_t)(b >> 6) * NC + c] |= 1ull << (b & 63);
        summ[(size_t)(b >> 12) * NC + c] |= 1ull << ((b >> 6) & 63);
        ++bsize[c];
    };
    auto del = [&](int c, int b) {
        uint64_t &w = bits[(size_t)(b >> 6) * NC + c];
        w &= ~(1ull << (b & 63));
        if (!w) summ[(size_t)(b >> 12) * NC + c] &= ~(1ull << ((b >> 6) & 63));
        --bsize[c];
    };
    for (int b = 0; b < nb; ++b)
        if (cnt[b] >= 0) add(cnt[b], b);
    // blocks taken in the current phase are marked in the count array itself
    // (kTaken, above every pending count; set to -1 by the commit), so the
    // clash test reads the count lines the commit touches next anyway
    const CT kTaken = std::numeric_limits<CT>::max();
    ptr.assign(1, 0);
    blocks.clear();
    blocks.reserve(pending);
    std::vector<int32_t> batch;
    const bool prof = getenv("FSE_PLAN_TIMING") != nullptr;
    double t_sel = 0.0, t_com = 0.0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    while (pending > 0) {
        const auto q0 = prof ? now() : std::chrono::steady_clock::time_point{};
        int nmin = 0;
        while (bsize[nmin] == 0) ++nmin;
        batch.clear();
        for (int sw = 0; sw < swords; ++sw) {
            uint64_t sm = summ[(size_t)sw * NC + nmin];
            while (sm) {
                const int w = (sw << 6) + __builtin_ctzll(sm);
                sm &= sm - 1;
                uint64_t m = bits[(size_t)w * NC + nmin];
                while (m) {
                    int b = (w << 6) + __builtin_ctzll(m);
                    m &= m - 1;
                    int r = b / cols, c = b - r * cols;
                    // only row-major-earlier neighbours can already be taken
                    bool clash = false;
                    if (c > 0 && cnt[b - 1] == kTaken) clash = true;
                    if (!clash && r > 0) {
                        int up = b - cols;
                        if (cnt[up] == kTaken || (c > 0 && cnt[up - 1] == kTaken) ||
                            (c + 1 < cols && cnt[up + 1] == kTaken))
                            clash = true;
                    }
                    if (clash) continue;
                    cnt[b] = kTaken;
                    batch.push_back(b);
                }
            }
        }
        const auto q1 = prof ? now() : std::chrono::steady_clock::time_point{};
        if (prof) t_sel += ms(q0, q1);
        for (int b : batch) {
            del(nmin, b);
            cnt[b] = -1;
            --pending;
        }
        // commit_batch (schedule.py:85-94): every neighbour's count drops by
        // one.  A pending block whose count falls below 0 is done from then on
        // (never selected: select_batch's pending set is counts >= 0); with
        // init_counts' counts that cannot happen (a pending count is at least
        // its number of pending lossy neighbours), with caller-supplied ones it
        // can, as in the reference.
        auto release = [&](int o) {
            if (cnt[o] >= 0) {
                del(cnt[o], o);
                if (--cnt[o] >= 0) add(cnt[o], o);
                else --pending;
            }
        };
        for (int b : batch) {
            int r = b / cols, c = b - r * cols;
            if (r > 0 && r + 1 < rows && c > 0 && c + 1 < cols) {  // interior: no bounds tests
                const int u = b - cols, d = b + cols;
                release(u - 1), release(u), release(u + 1), release(b - 1);
                release(b + 1), release(d - 1), release(d), release(d + 1);
                continue;
            }
            for (int dr = -1; dr <= 1; ++dr)
                for (int dc = -1; dc <= 1; ++dc) {
                    if (!dr && !dc) continue;
                    int rr = r + dr, cc = c + dc;
                    if (rr < 0 || rr >= rows || cc < 0 || cc >= cols) continue;
                    release(rr * cols + cc);
                }
        }
        blocks.insert(blocks.end(), batch.begin(), batch.end());
        ptr.push_back((int32_t)blocks.size());
        if (prof) t_com += ms(q1, now());
    }
    if (prof) fprintf(stderr, "plan   schedule loop: select %.1f ms, commit %.1f ms\n", t_sel, t_com);
}

struct Geometry {
    int H, W, B, rows, cols, d;
    void block_rect(int b, int &r0, int &r1, int &c0, int &c1) const {
        int r = b / cols, c = b - r * cols;
        r0 = r * B;
        r1 = std::min(r0 + B, H);
        c0 = c * B;
        c1 = std::min(c0 + B, W);
    }
    void window_rect(int b, int &r0, int &r1, int &c0, int &c1) const {
        block_rect(b, r0, r1, c0, c1);
        r0 = std::max(0, r0 - d);
        c0 = std::max(0, c0 - d);
        r1 = std::min(H, r1 + d);
        c1 = std::min(W, c1 + d);
    }
};

// Dependency levels over the processing order: level(b) = 1 + max level over
// lower-rank blocks whose samples b's window covers.  The window of block
// (r, c) covers exactly the blocks within Chebyshev radius R = ceil(d / B)
// (clamped to the grid): its rows run from floor((rB - d)/B) = r - ceil(d/B)
// to floor((rB + B + d - 1)/B) = r + ceil(d/B).  The square max is separable:
// HL[r][c] = max of level over row r, columns c +- R, kept up to date as
// batches are committed; a query is 2R+1 reads of HL.  T = int16_t while the
// level count fits (half the cache footprint of int32).
template <typename T>
int level_pass(const Plan &P, int rows, int cols, int R, std::vector<int32_t> &level) {
    std::vector<T> HL((size_t)rows * cols, (T)-1);
    int n_levels = 0;
    const int n_batches = (int)P.batch_ptr.size() - 1;
    for (int k = 0; k < n_batches; ++k) {
        const int i0 = P.batch_ptr[k], i1 = P.batch_ptr[k + 1];
        for (int i = i0; i < i1; ++i) {  // a batch reads only earlier batches
            const int b = P.batch_blocks[i];
            const int r = b / cols, c = b - r * cols;
            int m = -1;
            for (int rr = std::max(0, r - R); rr <= std::min(rows - 1, r + R); ++rr)
                m = std::max(m, (int)HL[(size_t)rr * cols + c]);
            level[b] = m + 1;
            n_levels = std::max(n_levels, m + 2);
        }
        for (int i = i0; i < i1; ++i) {
            const int b = P.batch_blocks[i];
            const int r = b / cols, c = b - r * cols;
            T *row = &HL[(size_t)r * cols];
            const T lv = (T)level[b];
            for (int cc = std::max(0, c - R); cc <= std::min(cols - 1, c + R); ++cc)
                row[cc] = std::max(row[cc], lv);
        }
    }
    return n_levels;
}

// ---- host threads -------------------------------------------------------------

// Run fn(k) on threads k = 0..T-1 (k = 0 on the caller).
template <class Fn>
void run_threads(int T, Fn &&fn) {
    std::vector<std::thread> pool;
    pool.reserve(T > 1 ? T - 1 : 0);
    for (int k = 1; k < T; ++k) pool.emplace_back([&fn, k] { fn(k); });
    fn(0);
    for (auto &t : pool) t.join();
}

int usable_cpus() {
#ifdef __linux__
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, (int)CPU_COUNT(&set));
#endif
    return std::max(1, (int)std::thread::hardware_concurrency());
}

// Smallest band of block rows a plan thread owns: the band's first-row fix-up
// (below) then never reaches its last row in practice.
constexpr int kMinBandRows = 16;
// Grids below this many blocks are planned on one thread (thread start-up
// costs more than the work).
constexpr long kParallelMinBlocks = 1L << 16;

// Threads for one plan: requested (0 = FSE_PLAN_THREADS, else 3/4 of the
// usable CPUs, at most 16), at most one per kMinBandRows block rows.
// requested > 0 forces that many (tests; bands down to one row), else
// FSE_PLAN_THREADS or 3/4 of the usable CPUs, at most `cap`.
int plan_threads(int requested, int cap, int rows, long nb) {
    if (requested > 0) return std::max(1, std::min(requested, rows));
    // a quarter of the CPUs stays free: the band threads spin between
    // phases, so a preempted one stalls all (measured in the bench, 16 CPUs:
    // 1080p plan 29.7 ms on 16 threads vs 4.0 ms on 12, with the clock
    // sampler and the launch thread running)
    const char *e = getenv("FSE_PLAN_THREADS");
    const int cpus = usable_cpus();
    int T = e ? atoi(e) : std::min(16, std::max(1, cpus - cpus / 4));
    T = std::min(T, cap);
    if (nb < kParallelMinBlocks) T = 1;
    T = std::min(T, rows / kMinBandRows);
    return std::max(1, T);
}

// Degeneracy test of conceal.py:53-58 / fse.py:150-151 on the host: does block
// b's window (its state as of the block's phase) hold a sample of positive
// weight?  A samples always weigh rho^dist > 0; R samples weigh
// delta*rho^dist, > 0 iff delta > 0.  `written` marks blocks reconstructed by
// earlier phases.
struct Usable {
    const Geometry &G;
    const uint8_t *mask;
    const uint8_t *flag;     // bit 0 LOST, bit 1 RECONSTRUCTED, bit 2 other sample in the block
    const uint8_t *sok;      // usable whatever was written (window-covered A / R0 block)
    const uint8_t *written;  // block reconstructed by an earlier phase
    bool r_counts;           // delta > 0
    bool operator()(int b) const {
        if (sok[b]) return true;
        const int B = G.B, cols = G.cols, W = G.W;
        int wr0, wr1, wc0, wc1;
        G.window_rect(b, wr0, wr1, wc0, wc1);
        int br0 = wr0 / B, br1 = (wr1 - 1) / B, bc0 = wc0 / B, bc1 = (wc1 - 1) / B;
        for (int pass = 0; pass < 2; ++pass)  // cheap whole-block test first
            for (int rr = br0; rr <= br1; ++rr)
                for (int cc = bc0; cc <= bc1; ++cc) {
                    int o = rr * cols + cc;
                    int or0, or1, oc0, oc1;
                    G.block_rect(o, or0, or1, oc0, oc1);
                    bool inside = or0 >= wr0 && or1 <= wr1 && oc0 >= wc0 && oc1 <= wc1;
                    if (pass == 0) {
                        if (!inside) continue;
                        if (flag[o] & 4) return true;
                        if (r_counts && ((flag[o] & 2) || (written[o] && (flag[o] & 1)))) return true;
                    } else {
                        if (inside) continue;
                        int y0 = std::max(or0, wr0), y1 = std::min(or1, wr1);
                        int x0 = std::max(oc0, wc0), x1 = std::min(oc1, wc1);
                        for (int y = y0; y < y1; ++y)
                            for (int x = x0; x < x1; ++x) {
                                uint8_t s = mask[(size_t)y * W + x];
                                if (s != FSE_LOST && s != FSE_RECONSTRUCTED) return true;
                                if (r_counts && (s == FSE_RECONSTRUCTED || (s == FSE_LOST && written[o])))
                                    return true;
                            }
                    }
                }
        return false;
    }
};

// ---- band-parallel optimized order ---------------------------------------------
//
// Algorithm 1 (schedule.py:60-105), the snapshot/deferral rule
// (conceal.py:145-163) and the dependency levels in one pass over the phases,
// on T threads.  Thread k owns the counts, buckets, ranks and levels of a
// static band of block rows [s_k, s_k+1).  Per phase:
//   A  all-reduce of the bands' smallest pending counts: the phase's N_min
//      (dissemination rounds, no shared counter).  The previous phase's
//      results become visible (written flags, level rows).
//   select  select_batch's greedy row-major rule only looks at the row above
//      and the block to the left, and only candidates (pending blocks of count
//      N_min) can be taken.  So the selection splits exactly at any row whose
//      row above holds no candidate: thread k selects rows [b_k, b_k+1), b_k
//      the first such row at or below s_k (per-row bucket tallies make the test
//      O(1); a band without one merges into the band above for the phase).
//   C  barrier; commit_batch: each band applies the count releases that land
//      in its own rows (from every batch member within one row of them),
//      decides degeneracy (Usable) and queries its members' levels.
// Results are identical to the sequential path (tested for many thread counts).

// Dissemination barrier with a min all-reduce folded in (ceil(log2 T)
// rounds; round i: thread k posts to k + 2^i, waits for k - 2^i).  Epochs
// only grow, so a slot is never reset.
// A band thread that fails (std::bad_alloc) sets `abort`; threads waiting in a
// barrier see it and unwind too, so no thread waits forever.
struct PlanAborted {};

struct MinBarrier {
    struct alignas(64) Slot {
        std::atomic<uint64_t> v{0};  // epoch << 32 | value
    };
    std::atomic<bool> abort{false};
    int T, rounds;
    std::vector<Slot> slots;  // [epoch parity][thread][round]: a thread is never two epochs ahead
    explicit MinBarrier(int T_) : T(T_), rounds(0) {
        while ((1 << rounds) < T) ++rounds;
        slots = std::vector<Slot>((size_t)2 * T * std::max(1, rounds));
    }
    // returns the minimum of every thread's `val` of this epoch (epoch >= 1, increasing by 1)
    int allreduce_min(int k, uint32_t epoch, int val) {
        Slot *S = &slots[(size_t)(epoch & 1) * T * std::max(1, rounds)];
        for (int i = 0; i < rounds; ++i) {
            const int to = (k + (1 << i)) % T;
            S[(size_t)to * rounds + i].v.store(((uint64_t)epoch << 32) | (uint32_t)val, std::memory_order_release);
            const std::atomic<uint64_t> &mine = S[(size_t)k * rounds + i].v;
            uint64_t got;
            for (int spin = 0; ((got = mine.load(std::memory_order_acquire)) >> 32) < epoch; ++spin) {
                if (spin < 8192) {
#if defined(__x86_64__) || defined(__i386__)
                    __builtin_ia32_pause();
#endif
                } else {
                    if (abort.load(std::memory_order_relaxed)) throw PlanAborted{};
                    std::this_thread::yield();
                }
            }
            val = std::min(val, (int)(uint32_t)got);
        }
        return val;
    }
};

#ifndef FSE_PLAN_SOLO  // dev knob: solo threshold (band candidates at N_min); -1 = never
#define FSE_PLAN_SOLO 4
#endif
template <typename CT, typename HT>
struct BandPlanner {
    const Geometry &G;
    const int T, rows, cols, R;
    const int NC;
    const std::vector<int> &s;  // band k owns block rows [s[k], s[k+1])
    CT *cnt;
    const Usable &usable;
    uint8_t *written;
    HT *HL;
    int32_t *rank;
    int32_t *level;
    MinBarrier bar;
    static constexpr CT kTaken = std::numeric_limits<CT>::max();
    static constexpr int kNone = INT_MAX;

    struct alignas(64) Band {
        int r0 = 0, r1 = 0, base = 0, nblk = 0;
        uint32_t epoch = 0;                // barrier epochs passed
        std::vector<uint64_t> bits, summ;  // [word][count], summary [sword][count]
        std::vector<uint64_t> supr;        // [sword / 64][count]: non-empty summary words
        std::vector<long> bsize;
        std::vector<int32_t> sel, prev_ok, okb, okptr, deferred, rowbuf;
        std::vector<uint8_t> lastrow;  // own last row's taken flags after the speculative select
        int maxlev = -1;
        bool lastchanged = false;
        double wait_ms = 0.0, sel_ms = 0.0, fix_ms = 0.0, com_ms = 0.0;  // FSE_PLAN_TIMING
    };
    struct alignas(64) Flag {
        std::atomic<int> v{0};
    };
    std::vector<Band> bands;
    std::vector<Flag> spec_done;  // band k's lastrow of phase ph is published: spec_done[k] = ph + 1
    std::atomic<int> any_lastchanged{0};
    std::atomic<int> overflow{0};  // a level does not fit HT: the caller re-plans with int32
    int n_phases = 0;
    int solo_next = 0;  // phase after thread 0's solo stretch (read after the park barrier)
    // phases whose bands hold at most this many candidates each run solo
    static constexpr int kSoloMax = FSE_PLAN_SOLO;
    bool prof = false;

    BandPlanner(const Geometry &G_, int T_, int R_, int NC_, const std::vector<int> &s_, CT *cnt_, const Usable &u,
                uint8_t *wr, HT *hl, int32_t *rk, int32_t *lv)
        : G(G_), T(T_), rows(G_.rows), cols(G_.cols), R(R_), NC(NC_), s(s_), cnt(cnt_), usable(u), written(wr),
          HL(hl), rank(rk), level(lv), bar(T_), bands(T_), spec_done(T_) {}

    int sync_min(int k, int v) { return bar.allreduce_min(k, ++bands[k].epoch, v); }

    // bucket ops on band bd (b: global block index)
    void add(Band &bd, int c, int b) {
        const int l = b - bd.base;
        bd.bits[(size_t)(l >> 6) * NC + c] |= 1ull << (l & 63);
        bd.summ[(size_t)(l >> 12) * NC + c] |= 1ull << ((l >> 6) & 63);
        bd.supr[(size_t)(l >> 18) * NC + c] |= 1ull << ((l >> 12) & 63);
        ++bd.bsize[c];
    }
    void del(Band &bd, int c, int b) {
        const int l = b - bd.base;
        uint64_t &w = bd.bits[(size_t)(l >> 6) * NC + c];
        w &= ~(1ull << (l & 63));
        if (!w) {
            uint64_t &sw = bd.summ[(size_t)(l >> 12) * NC + c];
            sw &= ~(1ull << ((l >> 6) & 63));
            if (!sw) bd.supr[(size_t)(l >> 18) * NC + c] &= ~(1ull << ((l >> 12) & 63));
        }
        --bd.bsize[c];
    }
    // blocks of bucket c of band bd in ascending order, through the two summary levels
    template <class Fn>
    void scan_bucket(const Band &bd, int c, Fn &&fn) const {
        const int nsup = (int)(bd.supr.size() / NC);
        for (int u = 0; u < nsup; ++u) {
            uint64_t su = bd.supr[(size_t)u * NC + c];
            while (su) {
                const int sw = (u << 6) + __builtin_ctzll(su);
                su &= su - 1;
                uint64_t sm = bd.summ[(size_t)sw * NC + c];
                while (sm) {
                    const int w = (sw << 6) + __builtin_ctzll(sm);
                    sm &= sm - 1;
                    uint64_t m = bd.bits[(size_t)w * NC + c];
                    while (m) {
                        fn(bd.base + (w << 6) + __builtin_ctzll(m));
                        m &= m - 1;
                    }
                }
            }
        }
    }
    // blocks of bucket c in the global block range [lo, hi) of band bd, ascending
    template <class Fn>
    void scan_range(const Band &bd, int c, int lo, int hi, Fn &&fn) const {
        int l0 = lo - bd.base, l1 = hi - bd.base;
        for (int w = l0 >> 6; w <= ((l1 - 1) >> 6); ++w) {
            uint64_t m = bd.bits[(size_t)w * NC + c];
            if (w == (l0 >> 6)) m &= ~0ull << (l0 & 63);
            if (w == ((l1 - 1) >> 6) && ((l1 & 63) != 0)) m &= ~0ull >> (64 - (l1 & 63));
            while (m) {
                fn(bd.base + (w << 6) + __builtin_ctzll(m));
                m &= m - 1;
            }
        }
    }

    void init_band(int k) {
        Band &bd = bands[k];
        bd.r0 = s[k];
        bd.r1 = s[k + 1];
        bd.base = bd.r0 * cols;
        bd.nblk = (bd.r1 - bd.r0) * cols;
        const int words = (bd.nblk + 63) / 64, swords = (words + 63) / 64;
        bd.bits.assign((size_t)words * NC, 0);
        bd.summ.assign((size_t)swords * NC, 0);
        bd.supr.assign((size_t)((swords + 63) / 64) * NC, 0);
        bd.bsize.assign(NC, 0);
        bd.lastrow.assign(cols, 0);
        bd.okptr.assign(1, 0);
        for (int b = bd.base; b < bd.base + bd.nblk; ++b)
            if (cnt[b] >= 0) add(bd, cnt[b], b);
    }

    // greedy rule on row r of band bd with the taken flags `up(c)` of row r - 1;
    // applies the decisions to cnt and returns whether any changed
    template <class Up>
    bool redo_row(Band &bd, int nmin, int r, Up &&up) {
        bool changed = false;
        int last = -2;  // column of the previous taken block in this row
        scan_range(bd, nmin, r * cols, (r + 1) * cols, [&](int b) {
            const int c = b - r * cols;
            const bool take = last != c - 1 && !(c > 0 && up(c - 1)) && !up(c) && !(c + 1 < cols && up(c + 1));
            const bool was = cnt[b] == kTaken;
            if (take) last = c;
            if (take != was) {
                cnt[b] = take ? kTaken : (CT)nmin;
                changed = true;
            }
        });
        return changed;
    }

    // first-row fix-up of band k against the row above as `up` reports it;
    // cascades down while rows change, then rebuilds the changed prefix of sel
    template <class Up>
    void fixup(int k, int nmin, Up &&up0) {
        Band &bd = bands[k];
        int r = bd.r0;
        if (!redo_row(bd, nmin, r, up0)) return;
        int last_changed = r;
        while (r + 1 < bd.r1) {
            const int ra = r;
            auto up = [&](int c) { return cnt[(size_t)ra * cols + c] == kTaken; };
            ++r;
            if (!redo_row(bd, nmin, r, up)) break;
            last_changed = r;
        }
        if (last_changed == bd.r1 - 1) bd.lastchanged = true;
        // sel: entries of rows <= last_changed are rebuilt from the taken flags
        const int lim = (last_changed + 1) * cols;
        size_t keep = 0;
        while (keep < bd.sel.size() && bd.sel[keep] < lim) ++keep;
        bd.rowbuf.clear();
        scan_range(bd, nmin, bd.r0 * cols, lim, [&](int b) {
            if (cnt[b] == kTaken) bd.rowbuf.push_back(b);
        });
        bd.sel.erase(bd.sel.begin(), bd.sel.begin() + keep);
        bd.sel.insert(bd.sel.begin(), bd.rowbuf.begin(), bd.rowbuf.end());
    }

    void release(Band &bd, int o) {
        if (cnt[o] >= 0) {
            del(bd, cnt[o], o);
            if (--cnt[o] >= 0) add(bd, cnt[o], o);
        }
    }
    // releases of batch member b (row rb, column cb) that land in rows [lo, hi)
    void release_around(Band &bd, int b, int lo, int hi) {
        const int rb = b / cols, cb = b - rb * cols;
        for (int rr = std::max(lo, rb - 1); rr <= std::min(hi - 1, rb + 1); ++rr)
            for (int cc = std::max(0, cb - 1); cc <= std::min(cols - 1, cb + 1); ++cc)
                if (rr != rb || cc != cb) release(bd, rr * cols + cc);
    }

    void apply_prev(Band &bd) {
        for (int b : bd.prev_ok) {
            written[b] = 1;
            const int r = b / cols, c = b - r * cols;
            HT *row = &HL[(size_t)r * cols];
            const HT lv = (HT)level[b];
            for (int cc = std::max(0, c - R); cc <= std::min(cols - 1, c + R); ++cc) row[cc] = std::max(row[cc], lv);
        }
        bd.prev_ok.clear();
    }

    int owner_band(int r) const { return (int)(std::upper_bound(s.begin(), s.end(), r) - s.begin()) - 1; }

    // degeneracy, rank and level of band bd's members of phase ph
    // (conceal.py:145-163), in row-major order
    void finish_members(Band &bd, int ph) {
        for (int b : bd.sel) {
            if (!usable(b)) {
                bd.deferred.push_back(b);
                continue;
            }
            rank[b] = ph;
            const int r = b / cols, c = b - r * cols;
            int m = -1;
            for (int rr = std::max(0, r - R); rr <= std::min(rows - 1, r + R); ++rr)
                m = std::max(m, (int)HL[(size_t)rr * cols + c]);
            level[b] = m + 1;
            bd.maxlev = std::max(bd.maxlev, m + 1);
            if (m + 1 >= (int)std::numeric_limits<HT>::max()) overflow.store(1, std::memory_order_relaxed);
            bd.okb.push_back(b);
            bd.prev_ok.push_back(b);
        }
        bd.okptr.push_back((int32_t)bd.okb.size());
    }

    // smallest pending count over every band, and the largest band's number of
    // pending blocks at it (the solo test); kNone when nothing is pending
    int global_min(int &maxcand) const {
        int nm = kNone;
        for (const Band &o : bands)
            for (int c = 0; c < std::min(nm, NC); ++c)
                if (o.bsize[c]) {
                    nm = c;
                    break;
                }
        maxcand = 0;
        if (nm != kNone)
            for (const Band &o : bands) maxcand = std::max(maxcand, (int)o.bsize[nm]);
        return nm;
    }

    // One whole phase on thread 0 while the other band threads are parked:
    // select_batch over all rows in order, then commit_batch, degeneracy and
    // levels.  Used for the phases whose N_min bucket is tiny (most phases of
    // a large frame hold a handful of blocks): no synchronisation at all.
    void solo_phase(int ph, int nmin) {
        for (Band &o : bands) o.sel.clear();
        for (Band &o : bands) {
            if (!o.bsize[nmin]) continue;
            scan_bucket(o, nmin, [&](int b) {
                const int r = b / cols, c = b - r * cols;
                if (c > 0 && cnt[b - 1] == kTaken) return;
                if (r > 0) {
                    const int up = b - cols;
                    if (cnt[up] == kTaken || (c > 0 && cnt[up - 1] == kTaken) ||
                        (c + 1 < cols && cnt[up + 1] == kTaken))
                        return;
                }
                cnt[b] = kTaken;
                o.sel.push_back(b);
            });
        }
        for (Band &o : bands)
            for (int b : o.sel) {
                del(o, nmin, b);
                cnt[b] = -1;
            }
        for (Band &o : bands)
            for (int b : o.sel) {
                const int r = b / cols;
                const int q0 = owner_band(std::max(0, r - 1)), q1 = owner_band(std::min(rows - 1, r + 1));
                for (int q = q0; q <= q1; ++q) release_around(bands[q], b, bands[q].r0, bands[q].r1);
            }
        for (Band &o : bands) finish_members(o, ph);
    }

    void run(int k) {
        Band &bd = bands[k];
        init_band(k);
        using clock = std::chrono::steady_clock;
        auto tp = prof ? clock::now() : clock::time_point{};
        auto lapt = [&](double &acc) {
            if (!prof) return;
            auto n = clock::now();
            acc += std::chrono::duration<double, std::milli>(n - tp).count();
            tp = n;
        };
        for (int ph = 0;; ++ph) {
            // ---- A: the phase's N_min, and the largest band candidate count at
            // it (packed: count 0xFFFF - n in the low bits, so min picks it)
            int lm = kNone;
            for (int c = 0; c < NC; ++c)
                if (bd.bsize[c]) {
                    lm = c;
                    break;
                }
            const int key = lm == kNone ? kNone : (lm << 16) | (0xFFFF - (int)std::min<long>(bd.bsize[lm], 0xFFFF));
            lapt(bd.com_ms);
            const int red = sync_min(k, key);
            lapt(bd.wait_ms);
            if (red == kNone) {
                apply_prev(bd);
                if (k == 0) n_phases = ph;
                break;
            }
            const int nmin = red >> 16, maxcand = 0xFFFF - (red & 0xFFFF);
            if (maxcand <= kSoloMax) {
                // ---- a stretch of tiny phases on thread 0; the others park.
                // Thread 0 also applies every band's previous-phase results
                // (the owners skip it here, so nothing races its level queries)
                if (k == 0) {
                    int p = ph, nm = nmin, mc = maxcand;
                    for (;;) {
                        for (Band &o : bands) apply_prev(o);  // results of phase p - 1
                        solo_phase(p, nm);
                        ++p;
                        nm = global_min(mc);
                        if (nm == kNone || mc > kSoloMax) break;
                    }
                    solo_next = p;
                    lapt(bd.sel_ms);
                }
                sync_min(k, 0);
                lapt(bd.wait_ms);
                ph = solo_next - 1;
                continue;
            }
            apply_prev(bd);
            // ---- speculative select (select_batch, schedule.py:60-82)
            bd.sel.clear();
            bd.lastchanged = false;
            if (bd.bsize[nmin]) {
                const int swords = (int)(bd.summ.size() / NC);
                for (int sw = 0; sw < swords; ++sw) {
                    uint64_t sm = bd.summ[(size_t)sw * NC + nmin];
                    while (sm) {
                        const int w = (sw << 6) + __builtin_ctzll(sm);
                        sm &= sm - 1;
                        uint64_t m = bd.bits[(size_t)w * NC + nmin];
                        while (m) {
                            const int b = bd.base + (w << 6) + __builtin_ctzll(m);
                            m &= m - 1;
                            const int r = b / cols, c = b - r * cols;
                            if (c > 0 && cnt[b - 1] == kTaken) continue;
                            if (r > bd.r0) {
                                const int up = b - cols;
                                if (cnt[up] == kTaken || (c > 0 && cnt[up - 1] == kTaken) ||
                                    (c + 1 < cols && cnt[up + 1] == kTaken))
                                    continue;
                            }
                            cnt[b] = kTaken;
                            bd.sel.push_back(b);
                        }
                    }
                }
            }
            {
                const CT *lr = &cnt[(size_t)(bd.r1 - 1) * cols];
                for (int c = 0; c < cols; ++c) bd.lastrow[c] = lr[c] == kTaken;
            }
            spec_done[k].v.store(ph + 1, std::memory_order_release);
            lapt(bd.sel_ms);
            // ---- B: fix-up against the band above's speculative last row
            // (a point-to-point wait: those rows depend on nothing else)
            if (k > 0 && bd.bsize[nmin]) {
                const std::atomic<int> &f = spec_done[k - 1].v;
                for (int spin = 0; f.load(std::memory_order_acquire) < ph + 1; ++spin)
                    if (spin > 8192) {
                        if (bar.abort.load(std::memory_order_relaxed)) throw PlanAborted{};
                        std::this_thread::yield();
                    }
                lapt(bd.wait_ms);
                const uint8_t *up = bands[k - 1].lastrow.data();
                fixup(k, nmin, [up](int c) { return up[c] != 0; });
            }
            if (bd.lastchanged) any_lastchanged.store(1, std::memory_order_relaxed);
            lapt(bd.fix_ms);
            sync_min(k, 0);  // ---- C
            lapt(bd.wait_ms);
            if (any_lastchanged.load(std::memory_order_relaxed)) {
                // a fix-up reached a band's last row, so the band below fixed
                // up against a stale row: redo every band's fix-up in band
                // order against the final row above (rare)
                sync_min(k, 0);
                if (k == 0) {
                    for (int q = 1; q < T; ++q) {
                        const int ra = bands[q].r0 - 1;
                        fixup(q, nmin, [&](int c) { return cnt[(size_t)ra * cols + c] == kTaken; });
                    }
                    any_lastchanged.store(0, std::memory_order_relaxed);
                }
                sync_min(k, 0);
            }
            // ---- commit_batch (schedule.py:85-94): own members done, then the
            // releases landing in own rows (own members, the band above's on
            // its last row, the band below's on its first row)
            for (int b : bd.sel) {
                del(bd, nmin, b);
                cnt[b] = -1;
            }
            for (int b : bd.sel) release_around(bd, b, bd.r0, bd.r1);
            if (k > 0) {
                const auto &sl = bands[k - 1].sel;
                for (size_t i = sl.size(); i-- > 0 && sl[i] >= bd.base - cols;) release_around(bd, sl[i], bd.r0, bd.r1);
            }
            if (k + 1 < T) {
                const auto &sl = bands[k + 1].sel;
                const int lim = bands[k + 1].base + cols;
                for (size_t i = 0; i < sl.size() && sl[i] < lim; ++i) release_around(bd, sl[i], bd.r0, bd.r1);
            }
            // ---- snapshot + degeneracy (conceal.py:145-163) and level queries
            finish_members(bd, ph);
        }
    }
};

// Per-block presence flags (only "any" is ever needed) of block rows [r0, r1):
// bit 0 a LOST sample (lost_per_block > 0, grid.py:138-144), bit 1 a
// RECONSTRUCTED sample, bit 2 any other state (class A, grid.py:124-130).
// Rows are scanned 8 bytes at a time; all-KNOWN and all-LOST words (the common
// cases) set one bit of their blocks without a per-byte pass.
void block_flags(const uint8_t *mask, int H, int W, int B, int cols, int r0, int r1, uint8_t *flag) {
    uint8_t lut[256];
    for (int v = 0; v < 256; ++v) lut[v] = v == FSE_LOST ? 1 : (v == FSE_RECONSTRUCTED ? 2 : 4);
    for (int y = r0 * B; y < std::min(H, r1 * B); ++y) {
        const uint8_t *row = mask + (size_t)y * W;
        uint8_t *fr = &flag[(size_t)(y / B) * cols];
        int x = 0;
        for (; x + 8 <= W; x += 8) {
            uint64_t w8;
            std::memcpy(&w8, row + x, 8);
            if (w8 == 0) {
                for (int c = x / B; c <= (x + 7) / B; ++c) fr[c] |= 4;
            } else if (w8 == 0x0101010101010101ull) {  // a run of LOST samples
                for (int c = x / B; c <= (x + 7) / B; ++c) fr[c] |= 1;
            } else {
                for (int i = 0; i < 8; ++i) fr[(x + i) / B] |= lut[row[x + i]];
            }
        }
        for (; x < W; ++x) fr[x / B] |= lut[row[x]];
    }
}

// "usable whatever was written" of the lossy blocks of block rows [ra, rb): a
// block lying wholly inside the window that holds an A sample (or, with
// delta > 0, a pre-reconstructed sample) makes the window usable.  The fully
// covered block range of block (r, c)'s window is [ilo(r), ihi(r)] x
// [jlo(c), jhi(c)], both monotone in their argument, so one row-major sweep
// with vertical running counts per column and a prefix count along the row
// answers every block in O(1).
void sure_usable(const Geometry &G, const uint8_t *flag, const uint8_t *lossy, bool r_counts, int ra, int rb,
                 uint8_t *sok) {
    const int B = G.B, rows = G.rows, cols = G.cols, d = G.d;
    auto lo_hi = [&](int i, int n, int S, int &lo, int &hi) {  // block i of n along an axis of S samples
        const int s0 = std::max(0, i * B - d);
        const int s1 = std::min(S, std::min(i * B + B, S) + d);
        lo = (s0 + B - 1) / B;
        hi = s1 == S ? n - 1 : s1 / B - 1;
    };
    auto good = [&](int o) { return (flag[o] & 4) || (r_counts && (flag[o] & 2)); };
    std::vector<int> jlo(cols), jhi(cols);
    for (int c = 0; c < cols; ++c) lo_hi(c, cols, G.W, jlo[c], jhi[c]);
    std::vector<int32_t> vcnt(cols, 0), pre(cols + 1, 0);
    int cur_lo = -1, cur_hi = -2;  // block rows summed into vcnt
    for (int r = ra; r < rb; ++r) {
        int ilo, ihi;
        lo_hi(r, rows, G.H, ilo, ihi);
        if (ilo > ihi) continue;
        if (cur_lo < 0) cur_lo = ilo, cur_hi = ilo - 1;
        while (cur_hi < ihi) {
            ++cur_hi;
            for (int c = 0; c < cols; ++c) vcnt[c] += good(cur_hi * cols + c) ? 1 : 0;
        }
        while (cur_lo < ilo) {
            for (int c = 0; c < cols; ++c) vcnt[c] -= good(cur_lo * cols + c) ? 1 : 0;
            ++cur_lo;
        }
        for (int c = 0; c < cols; ++c) pre[c + 1] = pre[c] + (vcnt[c] > 0 ? 1 : 0);
        for (int c = 0; c < cols; ++c) {
            const int b = r * cols + c;
            if (lossy[b] && jlo[c] <= jhi[c]) sok[b] = pre[jhi[c] + 1] - pre[jlo[c]] > 0 ? 1 : 0;
        }
    }
}

// init_counts (schedule.py:28-57) of block rows [ra, rb)
template <typename OutT>
void init_counts_rows(const uint8_t *lossy, int rows, int cols, int ra, int rb, OutT *counts) {
    auto h3 = [&](int r, int c) -> int {
        if (r < 0 || r >= rows) return 0;
        const uint8_t *p = lossy + (size_t)r * cols;
        return (c > 0 && p[c - 1] ? 1 : 0) + (p[c] ? 1 : 0) + (c + 1 < cols && p[c + 1] ? 1 : 0);
    };
    for (int r = ra; r < rb; ++r) {
        const int er = (r == 0) + (r == rows - 1);
        for (int c = 0; c < cols; ++c) {
            const int self = lossy[(size_t)r * cols + c] ? 1 : 0;
            if (!self) {
                counts[(size_t)r * cols + c] = -1;
                continue;
            }
            int n = h3(r - 1, c) + h3(r, c) + h3(r + 1, c) - 1;
            const int edges = er + (c == 0) + (c == cols - 1);
            if (edges == 1) n += kMarginBonus;
            else if (edges >= 2) n += kCornerBonus;
            counts[(size_t)r * cols + c] = (OutT)n;
        }
    }
}

// Level CSR from the per-block levels (row-major within a level).
void level_csr(Plan &P, const std::vector<int32_t> &level, int n_levels) {
    P.level_ptr.assign(n_levels + 1, 0);
    for (int b : P.batch_blocks) ++P.level_ptr[level[b] + 1];
    for (int l = 0; l < n_levels; ++l) P.level_ptr[l + 1] += P.level_ptr[l];
    P.level_blocks.assign(P.n_processed, 0);
    std::vector<int32_t> fill(P.level_ptr.begin(), P.level_ptr.end() - 1);
    const int nb = (int)level.size();
    for (int b = 0; b < nb; ++b)
        if (level[b] >= 0) P.level_blocks[fill[level[b]]++] = b;
}

// Level balancing (a pure re-leveling: ranks, batches and results unchanged).
// level_pass puts every block at its EARLIEST level, which leaves a frame with a
// few very wide first levels and a long tail of levels of a handful of windows
// (1080p, 30% isolated losses: 3,356 ... 1 windows over 101 levels), each tail
// level costing a lone window's latency with the GPU nearly empty.  A block may
// run at any level between its earliest one and one below its earliest
// DEPENDENT (a higher-rank block whose window covers it); blocks of a level
// never read each other with nonzero weight whatever their ranks (a lower-rank
// block sees a higher-rank one as lost), so only these true dependences order
// the launches.  Walking the batches from last to first (every dependent of a
// block lies in a later batch and is placed before it), a block of a level wider
// than max(narrow, wave) moves to the latest level within its slack that still
// has free slots: slots up to `narrow` in levels that stay on the one-window-
// per-SM kernel and, with wave > 0, up to `wave` in levels of at most one wave.
// The slack bound uses the same separable (2R+1)^2 minimum as level_pass's
// maximum.
int rebalance_levels(Plan &P, int narrow, int wave) {
    const int n_levels = (int)P.level_ptr.size() - 1;
    const int rows = P.rows, cols = P.cols;
    if (n_levels < 3 || narrow < 1 || rows < 1 || cols < 1) return 0;
    const int R = (P.d + P.B - 1) / P.B;
    const int nb = rows * cols;
    std::vector<int32_t> level(nb, -1);
    // cap: how many windows a level may hold after accepting blocks: `narrow`
    // while it stays that narrow, `wave` (if given) for a level of at most one
    // wave; wider levels accept nothing.  shed: how many blocks a level may give
    // away: any of them, down to `keep` = max(narrow, wave) windows (a level that
    // accepts gives nothing away).
    const int keep = std::max(narrow, wave);
    std::vector<int32_t> load(n_levels, 0), cap(n_levels, 0), shed(n_levels, 0);
    for (int l = 0; l < n_levels; ++l) {
        load[l] = P.level_ptr[l + 1] - P.level_ptr[l];
        for (int i = P.level_ptr[l]; i < P.level_ptr[l + 1]; ++i) level[P.level_blocks[i]] = l;
        if (load[l] <= narrow) cap[l] = narrow;
        else if (load[l] <= wave) cap[l] = wave;
        else cap[l] = load[l];
        shed[l] = load[l] > keep ? load[l] - keep : 0;
    }
    // latest level <= l with a free slot (union-find over full levels; -1 = none)
    std::vector<int32_t> nf(n_levels + 1);
    for (int l = 0; l <= n_levels; ++l) nf[l] = l;  // index l + 1 stands for level l, index 0 = none
    auto full = [&](int l) { return load[l] >= cap[l]; };
    std::function<int(int)> find = [&](int i) {
        while (nf[i] != i) {
            nf[i] = nf[nf[i]];
            i = nf[i];
        }
        return i;
    };
    for (int l = 0; l < n_levels; ++l)
        if (full(l)) nf[l + 1] = l;  // points to the previous index
    const int32_t kNone = INT32_MAX;
    std::vector<int32_t> HM((size_t)rows * cols, kNone);  // min new level of later-batch blocks over row r, columns c +- R
    const int n_batches = (int)P.batch_ptr.size() - 1;
    int moved = 0;
    int64_t free_slots = 0;  // the pass ends when every accepting level is full
    for (int l = 0; l < n_levels; ++l) free_slots += std::max(0, cap[l] - load[l]);
    for (int k = n_batches - 1; k >= 0 && free_slots > 0; --k) {
        const int i0 = P.batch_ptr[k], i1 = P.batch_ptr[k + 1];
        for (int i = i0; i < i1; ++i) {
            const int b = P.batch_blocks[i];
            const int lb = level[b];
            if (lb < 0 || shed[lb] <= 0) continue;  // its level gives nothing (more) away
            const int r = b / cols, c = b - r * cols;
            int32_t m = kNone;
            for (int rr = std::max(0, r - R); rr <= std::min(rows - 1, r + R); ++rr)
                m = std::min(m, HM[(size_t)rr * cols + c]);
            const int ub = (m == kNone ? n_levels : m) - 1;  // latest level b may run at
            if (ub <= lb) continue;
            const int t = find(ub + 1) - 1;  // latest level <= ub with a free slot
            if (t <= lb) continue;
            --load[lb];
            --shed[lb];
            ++load[t];
            --free_slots;
            if (full(t)) nf[t + 1] = t;
            level[b] = t;
            ++moved;
        }
        for (int i = i0; i < i1; ++i) {
            const int b = P.batch_blocks[i];
            if (level[b] < 0) continue;
            const int r = b / cols, c = b - r * cols;
            int32_t *row = &HM[(size_t)r * cols];
            const int32_t lv = level[b];
            for (int cc = std::max(0, c - R); cc <= std::min(cols - 1, c + R); ++cc) row[cc] = std::min(row[cc], lv);
        }
    }
    if (moved) level_csr(P, level, n_levels);
    return moved;
}

// Retry sweeps (conceal.py:69-94): sequential, row-major, each sees the
// previous results; every retried block is its own batch.  Levels of retried
// blocks continue the level rows HL.
template <typename HT>
int retry_sweeps(Plan &P, const Usable &usable, uint8_t *written, std::vector<int32_t> deferred, int n_phases,
                 HT *HL, int32_t *level, int R, int n_levels) {
    const int rows = P.rows, cols = P.cols;
    std::sort(deferred.begin(), deferred.end());
    std::vector<int32_t> pending = deferred, still;
    int next_rank = n_phases;
    for (int sweep = 0; sweep < std::max(rows, cols); ++sweep) {
        if (pending.empty()) break;
        still.clear();
        for (int b : pending) {
            if (usable(b)) {
                P.rank[b] = next_rank++;
                written[b] = 1;
                P.batch_blocks.push_back(b);
                P.batch_ptr.push_back((int32_t)P.batch_blocks.size());
                const int r = b / cols, c = b - r * cols;
                int m = -1;
                for (int rr = std::max(0, r - R); rr <= std::min(rows - 1, r + R); ++rr)
                    m = std::max(m, (int)HL[(size_t)rr * cols + c]);
                level[b] = m + 1;
                n_levels = std::max(n_levels, m + 2);
                HT *row = &HL[(size_t)r * cols];
                for (int cc = std::max(0, c - R); cc <= std::min(cols - 1, c + R); ++cc)
                    row[cc] = std::max(row[cc], (HT)(m + 1));
            } else {
                still.push_back(b);
            }
        }
        if (still.size() == pending.size()) break;
        pending.swap(still);
    }
    P.unconcealed = pending;
    P.n_processed = (int32_t)P.batch_blocks.size();
    return n_levels;
}

template <class T>
struct RawBuf {  // uninitialised array (filled by the band threads)
    std::unique_ptr<T[]> p;
    explicit RawBuf(size_t n) : p(new T[n]) {}
    T *get() const { return p.get(); }
};

// Band-parallel plan of the optimized order (see BandPlanner): every stage runs
// on the T band threads, the few sequential steps (band boundaries, batch
// offsets, retry sweeps, level offsets) on thread 0 between barriers.
// Returns false when a level does not fit HT.
template <typename CT, typename HT>
bool plan_optimized_parallel(Plan &P, const Geometry &G, int T, const uint8_t *mask, bool r_counts, bool prof) {
    const int rows = G.rows, cols = G.cols, nb = rows * cols, H = G.H, W = G.W, B = G.B;
    const int R = (G.d + B - 1) / B;
    constexpr int NC = 8 + kCornerBonus + 1;  // init_counts' counts are <= 8 + 5
    auto clk = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = clk();
    std::chrono::steady_clock::time_point t1, t2, t3;
    RawBuf<uint8_t> flag(nb), lossy(nb), sok(nb), written(nb);
    RawBuf<CT> cnt(nb);
    RawBuf<HT> HL(nb);
    RawBuf<int32_t> level(nb);
    std::vector<int> even(T + 1), s(T + 1), rowlossy(rows);
    for (int k = 0; k <= T; ++k) even[k] = (int)((long)rows * k / T);
    P.rank.assign(nb, INT32_MAX);
    Usable usable{G, mask, flag.get(), sok.get(), written.get(), r_counts};
    BandPlanner<CT, HT> bp(G, T, R, NC, s, cnt.get(), usable, written.get(), HL.get(), P.rank.data(), level.get());
    bp.prof = prof;
    bool ok = true;
    std::vector<int64_t> bofs, lofs;  // batch / level offsets per (phase or level, band)
    int n_levels = 0;
    std::atomic<bool> failed{false};
    run_threads(T, [&](int k) {
      try {
        // ---- per-block tallies of even bands (grid.py:138-144)
        {
            const int ra = even[k], rb = even[k + 1];
            std::memset(flag.get() + (size_t)ra * cols, 0, (size_t)(rb - ra) * cols);
            block_flags(mask, H, W, B, cols, ra, rb, flag.get());
            for (int r = ra; r < rb; ++r) {
                int n = 0;
                for (int b = r * cols; b < (r + 1) * cols; ++b) n += (lossy.get()[b] = flag.get()[b] & 1);
                rowlossy[r] = n;
            }
        }
        bp.sync_min(k, 0);
        if (k == 0) {
            // bands of equal lossy-block count, at least one row each
            std::vector<long> pre(rows + 1, 0);
            for (int r = 0; r < rows; ++r) pre[r + 1] = pre[r] + rowlossy[r];
            P.n_lossy = (int32_t)pre[rows];
            s[0] = 0;
            for (int q = 1; q < T; ++q) {
                const long target = pre[rows] * q / T;
                int r = (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
                s[q] = std::min(std::max(r, s[q - 1] + 1), rows - (T - q));
            }
            s[T] = rows;
        }
        bp.sync_min(k, 0);
        // ---- own rows: counts (schedule.py:28-57), sure-usable flags, level rows
        {
            const int ra = s[k], rb = s[k + 1];
            const size_t o = (size_t)ra * cols, n = (size_t)(rb - ra) * cols;
            std::memset(sok.get() + o, 0, n);
            std::memset(written.get() + o, 0, n);
            std::fill(HL.get() + o, HL.get() + o + n, (HT)-1);
            std::fill(level.get() + o, level.get() + o + n, -1);
            init_counts_rows(lossy.get(), rows, cols, ra, rb, cnt.get());
            sure_usable(G, flag.get(), lossy.get(), r_counts, ra, rb, sok.get());
        }
        // ---- the phases (the first all-reduce also orders the inits above)
        bp.run(k);
        bp.sync_min(k, 0);
        if (k == 0) {
            t1 = clk();
            ok = !bp.overflow.load();
            // batches: phase by phase, bands in order (row-major within a phase)
            const int nph = bp.n_phases;
            bofs.assign((size_t)nph * T + 1, 0);
            P.batch_ptr.assign(1, 0);
            int64_t run = 0;
            for (int ph = 0; ph < nph; ++ph) {
                const int64_t before = run;
                for (int q = 0; q < T; ++q) {
                    bofs[(size_t)ph * T + q] = run;
                    run += bp.bands[q].okptr[ph + 1] - bp.bands[q].okptr[ph];
                }
                if (run != before) P.batch_ptr.push_back((int32_t)run);
            }
            P.batch_blocks.resize(run);
        }
        if (!bp.sync_min(k, k == 0 ? (ok ? 1 : 0) : 1)) return;
        {
            const auto &bd = bp.bands[k];
            for (int ph = 0; ph < bp.n_phases; ++ph)
                std::copy(bd.okb.begin() + bd.okptr[ph], bd.okb.begin() + bd.okptr[ph + 1],
                          P.batch_blocks.begin() + bofs[(size_t)ph * T + k]);
        }
        bp.sync_min(k, 0);
        if (k == 0) {
            t2 = clk();
            std::vector<int32_t> deferred;
            for (auto &bd : bp.bands) {
                n_levels = std::max(n_levels, bd.maxlev + 1);
                deferred.insert(deferred.end(), bd.deferred.begin(), bd.deferred.end());
            }
            n_levels = retry_sweeps<HT>(P, usable, written.get(), std::move(deferred), bp.n_phases, HL.get(),
                                         level.get(), R, n_levels);
            lofs.assign((size_t)n_levels * T, 0);
            t3 = clk();
        }
        bp.sync_min(k, 0);
        // ---- level CSR (row-major within a level): counts per (level, band),
        // offsets, then every band places its own blocks
        const int32_t *lv = level.get();
        const int ra = s[k], rb = s[k + 1];
        std::vector<int64_t> mine(n_levels, 0);
        for (int b = ra * cols; b < rb * cols; ++b)
            if (lv[b] >= 0) ++mine[lv[b]];
        for (int l = 0; l < n_levels; ++l) lofs[(size_t)l * T + k] = mine[l];
        bp.sync_min(k, 0);
        if (k == 0) {
            P.level_ptr.assign(n_levels + 1, 0);
            int64_t run = 0;
            for (int l = 0; l < n_levels; ++l) {
                for (int q = 0; q < T; ++q) {
                    const int64_t c = lofs[(size_t)l * T + q];
                    lofs[(size_t)l * T + q] = run;
                    run += c;
                }
                P.level_ptr[l + 1] = (int32_t)run;
            }
            P.level_blocks.assign(run, 0);
        }
        bp.sync_min(k, 0);
        for (int l = 0; l < n_levels; ++l) mine[l] = lofs[(size_t)l * T + k];
        int32_t *out = P.level_blocks.data();
        for (int b = ra * cols; b < rb * cols; ++b)
            if (lv[b] >= 0) out[mine[lv[b]]++] = b;
      } catch (const PlanAborted &) {
      } catch (...) {  // std::bad_alloc: unwind every band thread
        failed.store(true);
        bp.bar.abort.store(true);
      }
    });
    if (failed.load()) throw std::bad_alloc();
    if (!ok) return false;
    if (prof) {
        const auto t4 = clk();
        fprintf(stderr, "plan   %d threads: tallies+phases %.1f ms, merge %.1f ms, retry %.1f ms, level csr %.1f ms\n", T,
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
        for (int k = 0; k < T; ++k)
            fprintf(stderr, "plan     band %d: wait %.1f select %.1f fixup %.1f commit %.1f ms\n", k, bp.bands[k].wait_ms,
                    bp.bands[k].sel_ms, bp.bands[k].fix_ms, bp.bands[k].com_ms);
    }
    return true;
}

int build_one(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p, int32_t order, Plan &P,
              int n_threads, int cap = 1 << 20) {
    int rc = validate(p, H, W, order);
    if (rc) return rc;
    Geometry G{H, W, p->block_size, (H + p->block_size - 1) / p->block_size,
               (W + p->block_size - 1) / p->block_size, p->d};
    const int rows = G.rows, cols = G.cols, nb = rows * cols, B = G.B;
    P.H = H; P.W = W; P.B = B; P.rows = rows; P.cols = cols; P.d = p->d; P.order = order;
    P.iterations = p->iterations; P.fft1 = p->fft1; P.fft2 = p->fft2;
    P.rho = p->rho; P.delta = p->delta; P.gamma = p->gamma;
    const int T = order == FSE_ORDER_OPTIMIZED ? plan_threads(n_threads, cap, rows, nb) : 1;
    const bool prof = getenv("FSE_PLAN_TIMING") != nullptr;
    const bool r_counts = p->delta > 0.0;
    P.max_wr = std::min(H, B + 2 * p->d);
    P.max_wc = std::min(W, B + 2 * p->d);
    auto clk = [] { return std::chrono::steady_clock::now(); };
    auto t_start = clk();
    auto lap = [&](const char *what) {
        if (!prof) return;
        auto now = clk();
        fprintf(stderr, "plan %-12s %.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t_start).count());
        t_start = now;
    };
    if (T > 1) {
        // level rows in int16 (half the cache footprint) unless a level
        // reaches 32767: then again in int32
        if (!plan_optimized_parallel<int8_t, int16_t>(P, G, T, mask, r_counts, prof))
            plan_optimized_parallel<int8_t, int32_t>(P, G, T, mask, r_counts, prof);
        lap("parallel");
        return FSE_OK;
    }
    std::vector<uint8_t> flag(nb, 0), lossy(nb), sok(nb, 0);
    std::vector<int32_t> counts;
    if (order == FSE_ORDER_OPTIMIZED) counts.resize(nb);
    block_flags(mask, H, W, B, cols, 0, rows, flag.data());
    P.n_lossy = 0;
    for (int b = 0; b < nb; ++b) {
        lossy[b] = flag[b] & 1;
        P.n_lossy += lossy[b];
    }
    lap("tallies");
    if (order == FSE_ORDER_OPTIMIZED) init_counts_rows(lossy.data(), rows, cols, 0, rows, counts.data());
    sure_usable(G, flag.data(), lossy.data(), r_counts, 0, rows, sok.data());
    lap("init_counts");
    std::vector<uint8_t> written(nb, 0);
    Usable usable{G, mask, flag.data(), sok.data(), written.data(), r_counts};

    // ---- one thread: processing phases in reference order
    std::vector<int32_t> ph_ptr, ph_blocks;
    if (order == FSE_ORDER_OPTIMIZED) {
        rc = schedule_impl(counts.data(), rows, cols, ph_ptr, ph_blocks);
        if (rc) return rc;
    } else {
        ph_ptr.assign(1, 0);
        for (int b = 0; b < nb; ++b)
            if (lossy[b]) {
                ph_blocks.push_back(b);
                ph_ptr.push_back((int32_t)ph_blocks.size());
            }
    }
    lap("schedule");
    P.rank.assign(nb, INT32_MAX);
    P.batch_ptr.assign(1, 0);
    P.batch_blocks.clear();
    std::vector<int32_t> deferred, ok;
    const int n_phases = (int)ph_ptr.size() - 1;
    for (int ph = 0; ph < n_phases; ++ph) {
        ok.clear();
        for (int i = ph_ptr[ph]; i < ph_ptr[ph + 1]; ++i) {
            int b = ph_blocks[i];
            if (usable(b)) ok.push_back(b);
            else deferred.push_back(b);
        }
        for (int b : ok) {  // writes land only after the whole batch (snapshot)
            P.rank[b] = ph;
            written[b] = 1;
        }
        if (!ok.empty()) {
            P.batch_blocks.insert(P.batch_blocks.end(), ok.begin(), ok.end());
            P.batch_ptr.push_back((int32_t)P.batch_blocks.size());
        }
    }
    // retry sweeps: sequential, row-major, each sees the previous results
    // (levels of the retried blocks come from the level pass below)
    {
        std::sort(deferred.begin(), deferred.end());
        std::vector<int32_t> pending = deferred, still;
        int next_rank = n_phases;
        for (int sweep = 0; sweep < std::max(rows, cols); ++sweep) {
            if (pending.empty()) break;
            still.clear();
            for (int b : pending) {
                if (usable(b)) {
                    P.rank[b] = next_rank++;
                    written[b] = 1;
                    P.batch_blocks.push_back(b);
                    P.batch_ptr.push_back((int32_t)P.batch_blocks.size());
                } else {
                    still.push_back(b);
                }
            }
            if (still.size() == pending.size()) break;
            pending.swap(still);
        }
        P.unconcealed = pending;
        P.n_processed = (int32_t)P.batch_blocks.size();
    }
    lap("ranks");
    // dependency levels over the processing order (level_pass)
    std::vector<int32_t> level(nb, -1);
    const int R = (p->d + B - 1) / B;
    const int n_batches = (int)P.batch_ptr.size() - 1;
    int n_levels = n_batches < 32000 ? level_pass<int16_t>(P, rows, cols, R, level)
                                     : level_pass<int32_t>(P, rows, cols, R, level);
    level_csr(P, level, n_levels);
    lap("levels");
    return FSE_OK;
}

}  // namespace
}  // namespace fse

using fse::fail;

extern "C" {

const char *fse_last_error(void) { return fse::g_last_error.c_str(); }

int fse_init_counts(const uint8_t *lossy, int32_t rows, int32_t cols, int32_t *counts) {
    if (!lossy || !counts || rows < 1 || cols < 1) return fail(FSE_EINVAL, "bad arguments");
    fse::init_counts_impl(lossy, rows, cols, counts);
    return FSE_OK;
}

int fse_schedule_all(const int32_t *counts, int32_t rows, int32_t cols, int32_t *ptr,
                     int32_t *blocks, int32_t *n_batches) {
    if (!counts || !ptr || !blocks || !n_batches || rows < 1 || cols < 1)
        return fail(FSE_EINVAL, "bad arguments");
    std::vector<int32_t> vp, vb;
    try {
        if (int rc = fse::schedule_impl(counts, rows, cols, vp, vb)) return rc;
    } catch (const std::exception &e) {
        return fail(FSE_ENOMEM, e.what());
    }
    std::memcpy(ptr, vp.data(), vp.size() * sizeof(int32_t));
    if (!vb.empty()) std::memcpy(blocks, vb.data(), vb.size() * sizeof(int32_t));
    *n_batches = (int32_t)vp.size() - 1;
    return FSE_OK;
}

static int plan_build(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p, int32_t order,
                      int32_t n_threads, int32_t cap, FsePlan **out) {
    if (!mask || !out) return fail(FSE_EINVAL, "mask/out is NULL");
    if (n_threads < 0) return fail(FSE_EINVAL, "n_threads must be >= 0");
    FsePlan *plan = nullptr;
    try {
        plan = new FsePlan();
        int rc = fse::build_one(mask, H, W, p, order, plan->p, n_threads, cap);
        if (rc) {
            delete plan;
            return rc;
        }
    } catch (const std::exception &e) {
        delete plan;
        return fail(FSE_ENOMEM, e.what());
    }
    *out = plan;
    return FSE_OK;
}

int fse_plan_build(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p,
                   int32_t order, FsePlan **out) {
    return plan_build(mask, H, W, p, order, 0, 1 << 20, out);
}

int fse_plan_build_threads(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p,
                           int32_t order, int32_t n_threads, FsePlan **out) {
    return plan_build(mask, H, W, p, order, n_threads, 1 << 20, out);
}

int fse_plan_build_many(int32_t n, const uint8_t *const *masks, int32_t H, int32_t W,
                        const FseParamsC *p, int32_t order, int32_t n_threads, FsePlan **out) {
    if (n < 0 || (n > 0 && (!masks || !out))) return fail(FSE_EINVAL, "bad arguments");
    // host threads: the caller's count, else FSE_PLAN_THREADS (set per local
    // rank under torchrun), else the usable CPUs (frames are independent: the
    // frame workers never wait on each other)
    int all = n_threads;
    if (all <= 0) {
        const char *e = getenv("FSE_PLAN_THREADS");
        all = e ? std::max(1, atoi(e)) : fse::usable_cpus();
    }
    int nt = std::max(1, std::min(all, n));
    std::vector<int> rcs(n, 0);
    std::vector<std::string> errs(n);
    std::atomic<int> next(0);
    // frames share the threads: each plan may use the band threads the frame
    // count leaves over (3/4 of them: band threads spin), one when frames >=
    // threads
    const int per_plan = std::max(1, (all - all / 4) / std::max(1, n));
    auto work = [&]() {
        for (int i; (i = next.fetch_add(1)) < n;) {
            out[i] = nullptr;
            rcs[i] = plan_build(masks[i], H, W, p, order, 0, per_plan, &out[i]);
            if (rcs[i]) errs[i] = fse_last_error();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &t : pool) t.join();
    for (int i = 0; i < n; ++i)
        if (rcs[i]) {
            for (int j = 0; j < n; ++j) {
                fse_plan_free(out[j]);
                out[j] = nullptr;
            }
            return fail(rcs[i], errs[i]);
        }
    return FSE_OK;
}

void fse_plan_free(FsePlan *plan) { delete plan; }

int fse_plan_sizes(const FsePlan *plan, int32_t *s) {
    if (!plan || !s) return fail(FSE_EINVAL, "NULL argument");
    const fse::Plan &P = plan->p;
    s[0] = P.rows;
    s[1] = P.cols;
    s[2] = P.n_lossy;
    s[3] = P.n_processed;
    s[4] = (int32_t)P.batch_ptr.size() - 1;
    s[5] = (int32_t)P.batch_blocks.size();
    s[6] = (int32_t)P.level_ptr.size() - 1;
    s[7] = (int32_t)P.unconcealed.size();
    s[8] = P.max_wr;
    s[9] = P.max_wc;
    return FSE_OK;
}

int fse_plan_batches(const FsePlan *plan, int32_t *ptr, int32_t *blocks) {
    if (!plan || !ptr || !blocks) return fail(FSE_EINVAL, "NULL argument");
    const fse::Plan &P = plan->p;
    std::copy(P.batch_ptr.begin(), P.batch_ptr.end(), ptr);
    std::copy(P.batch_blocks.begin(), P.batch_blocks.end(), blocks);
    return FSE_OK;
}

int fse_plan_levels(const FsePlan *plan, int32_t *ptr, int32_t *blocks) {
    if (!plan || !ptr || !blocks) return fail(FSE_EINVAL, "NULL argument");
    const fse::Plan &P = plan->p;
    std::copy(P.level_ptr.begin(), P.level_ptr.end(), ptr);
    std::copy(P.level_blocks.begin(), P.level_blocks.end(), blocks);
    return FSE_OK;
}

int fse_plan_rebalance(FsePlan *plan, int32_t narrow, int32_t wave, int32_t *moved) {
    if (!plan) return fail(FSE_EINVAL, "NULL plan");
    if (narrow < 0 || wave < 0) return fail(FSE_EINVAL, "narrow and wave must be >= 0");
    const int n = narrow > 0 ? fse::rebalance_levels(plan->p, narrow, wave) : 0;
    if (moved) *moved = n;
    return FSE_OK;
}

int fse_plan_ranks(const FsePlan *plan, int32_t *rank) {
    if (!plan || !rank) return fail(FSE_EINVAL, "NULL argument");
    std::copy(plan->p.rank.begin(), plan->p.rank.end(), rank);
    return FSE_OK;
}

int fse_plan_unconcealed(const FsePlan *plan, int32_t *blocks) {
    if (!plan || !blocks) return fail(FSE_EINVAL, "NULL argument");
    std::copy(plan->p.unconcealed.begin(), plan->p.unconcealed.end(), blocks);
    return FSE_OK;
}

// Serialised plan: int32 header, three doubles, then the rank table and the
// batch / level CSRs and the unconcealed list.  One rank plans a frame and
// broadcasts these bytes; the others import them (strips.py).
static const int32_t kPlanMagic = 0x46534550;  // "FSEP"
static const int kPlanHdr = 24;

int64_t fse_plan_export_size(const FsePlan *plan) {
    if (!plan) return fail(FSE_EINVAL, "NULL plan");
    const fse::Plan &P = plan->p;
    const size_t n = P.rank.size() + P.batch_ptr.size() + P.batch_blocks.size() + P.level_ptr.size() +
                     P.level_blocks.size() + P.unconcealed.size();
    return (int64_t)(kPlanHdr * sizeof(int32_t) + 3 * sizeof(double) + n * sizeof(int32_t));
}

int fse_plan_export(const FsePlan *plan, void *buf, int64_t size) {
    if (!plan || !buf) return fail(FSE_EINVAL, "NULL argument");
    if (size < fse_plan_export_size(plan)) return fail(FSE_EINVAL, "export buffer too small");
    const fse::Plan &P = plan->p;
    int32_t h[kPlanHdr] = {kPlanMagic, 1, P.H, P.W, P.B, P.rows, P.cols, P.d, P.order, P.iterations,
                           P.fft1, P.fft2, P.n_lossy, P.n_processed, P.max_wr, P.max_wc,
                           (int32_t)P.rank.size(), (int32_t)P.batch_ptr.size(), (int32_t)P.batch_blocks.size(),
                           (int32_t)P.level_ptr.size(), (int32_t)P.level_blocks.size(),
                           (int32_t)P.unconcealed.size(), 0, 0};
    unsigned char *o = static_cast<unsigned char *>(buf);
    auto put = [&](const void *src, size_t bytes) {
        if (bytes) std::memcpy(o, src, bytes);
        o += bytes;
    };
    put(h, sizeof(h));
    const double dd[3] = {P.rho, P.delta, P.gamma};
    put(dd, sizeof(dd));
    for (const std::vector<int32_t> *v : {&P.rank, &P.batch_ptr, &P.batch_blocks, &P.level_ptr, &P.level_blocks,
                                          &P.unconcealed})
        put(v->data(), v->size() * sizeof(int32_t));
    return FSE_OK;
}

int fse_plan_import(const void *buf, int64_t size, FsePlan **out) {
    if (!buf || !out) return fail(FSE_EINVAL, "NULL argument");
    if (size < (int64_t)(kPlanHdr * sizeof(int32_t) + 3 * sizeof(double))) return fail(FSE_EINVAL, "truncated plan");
    const unsigned char *in = static_cast<const unsigned char *>(buf);
    int32_t h[kPlanHdr];
    std::memcpy(h, in, sizeof(h));
    if (h[0] != kPlanMagic || h[1] != 1) return fail(FSE_EINVAL, "not a serialised plan");
    for (int i = 16; i < 22; ++i)
        if (h[i] < 0) return fail(FSE_EINVAL, "corrupt plan header");
    const int64_t need = (int64_t)(kPlanHdr * sizeof(int32_t) + 3 * sizeof(double)) +
                         (int64_t)sizeof(int32_t) * ((int64_t)h[16] + h[17] + h[18] + h[19] + h[20] + h[21]);
    if (size < need) return fail(FSE_EINVAL, "truncated plan");
    if ((int64_t)h[5] * h[6] != h[16] || h[17] < 1 || h[19] < 1) return fail(FSE_EINVAL, "inconsistent plan");
    FsePlan *plan = nullptr;
    try {
        plan = new FsePlan();
        fse::Plan &P = plan->p;
        P.H = h[2]; P.W = h[3]; P.B = h[4]; P.rows = h[5]; P.cols = h[6]; P.d = h[7]; P.order = h[8];
        P.iterations = h[9]; P.fft1 = h[10]; P.fft2 = h[11]; P.n_lossy = h[12]; P.n_processed = h[13];
        P.max_wr = h[14]; P.max_wc = h[15];
        in += sizeof(h);
        double dd[3];
        std::memcpy(dd, in, sizeof(dd));
        in += sizeof(dd);
        P.rho = dd[0]; P.delta = dd[1]; P.gamma = dd[2];
        int k = 16;
        for (std::vector<int32_t> *v : {&P.rank, &P.batch_ptr, &P.batch_blocks, &P.level_ptr, &P.level_blocks,
                                        &P.unconcealed}) {
            v->resize(h[k++]);
            if (!v->empty()) std::memcpy(v->data(), in, v->size() * sizeof(int32_t));
            in += v->size() * sizeof(int32_t);
        }
        if (P.batch_ptr.back() != (int32_t)P.batch_blocks.size() ||
            P.level_ptr.back() != (int32_t)P.level_blocks.size()) {
            delete plan;
            return fail(FSE_EINVAL, "inconsistent plan CSR");
        }
    } catch (const std::exception &e) {
        delete plan;
        return fail(FSE_ENOMEM, e.what());
    }
    *out = plan;
    return FSE_OK;
}

}  // extern "C"
