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
#include <atomic>
#include <climits>
#include <limits>
#include <cstring>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>

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

int build_one(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p, int32_t order,
              Plan &P) {
    int rc = validate(p, H, W, order);
    if (rc) return rc;
    Geometry G{H, W, p->block_size, (H + p->block_size - 1) / p->block_size,
               (W + p->block_size - 1) / p->block_size, p->d};
    const int rows = G.rows, cols = G.cols, nb = rows * cols, B = G.B;
    P.H = H; P.W = W; P.B = B; P.rows = rows; P.cols = cols; P.d = p->d; P.order = order;
    P.iterations = p->iterations; P.fft1 = p->fft1; P.fft2 = p->fft2;
    P.rho = p->rho; P.delta = p->delta; P.gamma = p->gamma;

    const bool prof = getenv("FSE_PLAN_TIMING") != nullptr;
    auto clk = [] { return std::chrono::steady_clock::now(); };
    auto t_start = clk();
    auto lap = [&](const char *what) {
        if (!prof) return;
        auto now = clk();
        fprintf(stderr, "plan %-12s %.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t_start).count());
        t_start = now;
    };
    // per-block presence flags (only "any" is ever needed): bit 0 a LOST sample
    // (lost_per_block > 0, grid.py:138-144), bit 1 a RECONSTRUCTED sample, bit 2
    // any other state (class A, grid.py:124-130).  Rows are scanned 8 bytes at a
    // time; all-KNOWN and all-LOST words (the common cases) set one bit of
    // their blocks without a per-byte pass.
    std::vector<uint8_t> flag(nb, 0);
    {
        uint8_t lut[256];
        for (int v = 0; v < 256; ++v) lut[v] = v == FSE_LOST ? 1 : (v == FSE_RECONSTRUCTED ? 2 : 4);
        for (int y = 0; y < H; ++y) {
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
    auto nL = [&](int b) { return (flag[b] & 1) != 0; };
    auto nR0 = [&](int b) { return (flag[b] & 2) != 0; };
    auto nA = [&](int b) { return (flag[b] & 4) != 0; };
    std::vector<uint8_t> lossy(nb);
    P.n_lossy = 0;
    for (int b = 0; b < nb; ++b) {
        lossy[b] = nL(b);
        P.n_lossy += lossy[b];
    }
    P.max_wr = std::min(H, B + 2 * p->d);
    P.max_wc = std::min(W, B + 2 * p->d);

    lap("tallies");
    // processing phases in reference order
    std::vector<int32_t> ph_ptr, ph_blocks;
    if (order == FSE_ORDER_OPTIMIZED) {
        std::vector<int32_t> counts(nb);
        init_counts_impl(lossy.data(), rows, cols, counts.data());
        lap("init_counts");
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
    // degeneracy (fse.py:150-151): no sample of positive weight.  A samples
    // always weigh rho^dist > 0; R samples weigh delta*rho^dist, > 0 iff delta > 0.
    std::vector<uint8_t> written(nb, 0);
    const bool r_counts = p->delta > 0.0;
    // Fast path: a block lying wholly inside the window that holds an A sample
    // (or, with delta > 0, a pre-reconstructed sample) makes the window usable
    // whatever was written since.  The fully covered block range of block
    // (r, c)'s window is [ilo(r), ihi(r)] x [jlo(c), jhi(c)], both monotone in
    // their argument, so one row-major sweep with vertical running counts per
    // column and a prefix count along the row answers every block in O(1).
    std::vector<uint8_t> sok(nb, 0);
    {
        auto lo_hi = [&](int i, int n, int S, int &lo, int &hi) {  // block i of n along an axis of S samples
            const int s0 = std::max(0, i * B - p->d);
            const int s1 = std::min(S, std::min(i * B + B, S) + p->d);
            lo = (s0 + B - 1) / B;
            hi = s1 == S ? n - 1 : s1 / B - 1;
        };
        std::vector<int> jlo(cols), jhi(cols);
        for (int c = 0; c < cols; ++c) lo_hi(c, cols, W, jlo[c], jhi[c]);
        std::vector<int32_t> vcnt(cols, 0), pre(cols + 1, 0);
        int cur_lo = 0, cur_hi = -1;  // block rows summed into vcnt
        for (int r = 0; r < rows; ++r) {
            int ilo, ihi;
            lo_hi(r, rows, H, ilo, ihi);
            if (ilo > ihi) continue;
            while (cur_hi < ihi) {
                ++cur_hi;
                for (int c = 0; c < cols; ++c) {
                    const int o = cur_hi * cols + c;
                    vcnt[c] += (nA(o) || (r_counts && nR0(o))) ? 1 : 0;
                }
            }
            while (cur_lo < ilo) {
                for (int c = 0; c < cols; ++c) {
                    const int o = cur_lo * cols + c;
                    vcnt[c] -= (nA(o) || (r_counts && nR0(o))) ? 1 : 0;
                }
                ++cur_lo;
            }
            for (int c = 0; c < cols; ++c) pre[c + 1] = pre[c] + (vcnt[c] > 0 ? 1 : 0);
            for (int c = 0; c < cols; ++c) {
                const int b = r * cols + c;
                if (lossy[b] && jlo[c] <= jhi[c]) sok[b] = pre[jhi[c] + 1] - pre[jlo[c]] > 0 ? 1 : 0;
            }
        }
    }
    auto usable = [&](int b) -> bool {
        if (sok[b]) return true;
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
                        if (nA(o)) return true;
                        if (r_counts && (nR0(o) || (written[o] && nL(o)))) return true;
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
    };

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

    lap("ranks");
    // dependency levels over the processing order (level_pass)
    std::vector<int32_t> level(nb, -1);
    const int R = (p->d + B - 1) / B;
    const int n_batches = (int)P.batch_ptr.size() - 1;
    int n_levels = n_batches < 32000 ? level_pass<int16_t>(P, rows, cols, R, level)
                                     : level_pass<int32_t>(P, rows, cols, R, level);
    P.level_ptr.assign(n_levels + 1, 0);
    for (int b : P.batch_blocks) ++P.level_ptr[level[b] + 1];
    for (int l = 0; l < n_levels; ++l) P.level_ptr[l + 1] += P.level_ptr[l];
    P.level_blocks.assign(P.n_processed, 0);
    std::vector<int32_t> fill(P.level_ptr.begin(), P.level_ptr.end() - 1);
    for (int b = 0; b < nb; ++b)  // row-major within a level
        if (level[b] >= 0) P.level_blocks[fill[level[b]]++] = b;
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

int fse_plan_build(const uint8_t *mask, int32_t H, int32_t W, const FseParamsC *p,
                   int32_t order, FsePlan **out) {
    if (!mask || !out) return fail(FSE_EINVAL, "mask/out is NULL");
    FsePlan *plan = nullptr;
    try {
        plan = new FsePlan();
        int rc = fse::build_one(mask, H, W, p, order, plan->p);
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

int fse_plan_build_many(int32_t n, const uint8_t *const *masks, int32_t H, int32_t W,
                        const FseParamsC *p, int32_t order, int32_t n_threads, FsePlan **out) {
    if (n < 0 || (n > 0 && (!masks || !out))) return fail(FSE_EINVAL, "bad arguments");
    int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    nt = std::max(1, std::min(nt, n));
    std::vector<int> rcs(n, 0);
    std::vector<std::string> errs(n);
    std::atomic<int> next(0);
    auto work = [&]() {
        for (int i; (i = next.fetch_add(1)) < n;) {
            out[i] = nullptr;
            rcs[i] = fse_plan_build(masks[i], H, W, p, order, &out[i]);
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

}  // extern "C"
