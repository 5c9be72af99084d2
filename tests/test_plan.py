"""Host side of the B200 path, CPU only: the C++ scheduler / plan in
libfse_b200.so against the reference's golden schedules and concealment
batches, and the level plan executed on the CPU (oracle kernel, rank-based
classification, racing write-back) against the reference's outputs."""

import os
import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2207_00233_b200 as P
from helpers import conceal_case, csr, emulate_levels
from oracle import oracle as O
from paper_2207_00233_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(REPO, "include", "fse_b200.h")).read()
    declared = set(re.findall(r"^(?:int|void|const char \*|int64_t)\s*\**(fse_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS)
    assert set(_lib.exports_present()) == declared


def resimulate(rows, cols, lossy):
    """Dict-based restatement of the wavefront order (reference tests/reference.py:74-119)."""
    def nbs(r, c):
        return [(r + a, c + b) for a in (-1, 0, 1) for b in (-1, 0, 1)
                if (a, b) != (0, 0) and 0 <= r + a < rows and 0 <= c + b < cols]
    cnt = {}
    for r in range(rows):
        for c in range(cols):
            if (r, c) not in lossy:
                cnt[(r, c)] = -1
                continue
            e = (r == 0) + (r == rows - 1) + (c == 0) + (c == cols - 1)
            cnt[(r, c)] = sum(x in lossy for x in nbs(r, c)) + (3 if e == 1 else 5 if e >= 2 else 0)
    out = []
    while any(v >= 0 for v in cnt.values()):
        m = min(v for v in cnt.values() if v >= 0)
        batch, taken = [], set()
        for r in range(rows):
            for c in range(cols):
                if cnt[(r, c)] == m and not any(x in taken for x in nbs(r, c)):
                    batch.append(r * cols + c)
                    taken.add((r, c))
        for b in batch:
            r, c = divmod(b, cols)
            cnt[(r, c)] = -1
            for x in nbs(r, c):
                cnt[x] -= 1
        out.append(batch)
    return out


def grid_of(rows, cols, B=8):
    return P.build_grid(cols * B, rows * B, B)


def test_scheduler_matches_reference_golden(golden):
    g = golden("schedule_cases.npz")
    for i in range(int(g["n_cases"])):
        t = g[f"s{i}_table"]
        grid = grid_of(*t.shape, B=4)
        c = P.init_counts(grid, t)
        np.testing.assert_array_equal(c, g[f"s{i}_counts"])
        assert P.schedule_all(grid, c) == csr(g[f"s{i}_ptr"], g[f"s{i}_blocks"])


def test_c1_scheduler_matches_resimulation_on_100_random_grids():
    rng = np.random.default_rng(0)
    for _ in range(100):
        rows, cols = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        table = (rng.uniform(size=(rows, cols)) < rng.uniform(0.05, 1.0)).astype(np.int64)
        grid = grid_of(rows, cols, 16)
        lossy = {(r, c) for r in range(rows) for c in range(cols) if table[r, c]}
        assert P.schedule_all(grid, P.init_counts(grid, table)) == resimulate(rows, cols, lossy)


def test_known_answers_3x3():
    grid = grid_of(3, 3)
    counts = P.init_counts(grid, np.ones((3, 3)))
    assert counts.tolist() == [8] * 9
    assert P.select_batch(grid, counts) == [0, 2, 6, 8]
    batches = P.schedule_all(grid, counts)
    assert batches == [[0, 2, 6, 8], [4], [1, 7], [3, 5]]
    P.commit_batch(grid, counts, [0, 2, 6, 8])
    assert counts.tolist() == [-1, 6, -1, 6, 4, 6, -1, 6, -1]
    P.commit_batch(grid, counts, [4])
    assert counts.tolist() == [-2, 5, -2, 5, -1, 5, -2, 5, -2]
    assert P.render_batch_trace(grid, batches) == "1 3 1\n4 2 4\n1 3 1"


def test_small_grids_and_empty():
    g1 = grid_of(1, 1)
    c = P.init_counts(g1, np.ones((1, 1)))
    assert c.tolist() == [5]
    assert P.schedule_all(g1, c) == [[0]]
    g = grid_of(4, 4)
    c = P.init_counts(g, np.zeros((4, 4)))
    assert (c == -1).all() and P.schedule_all(g, c) == []
    with pytest.raises(P.EmptyScheduleError):
        P.select_batch(g, c)
    g5 = grid_of(5, 5)
    t = np.zeros((5, 5)); t[2, 2] = 1
    c = P.init_counts(g5, t)
    assert c[12] == 0 and all(v == -1 for i, v in enumerate(c) if i != 12)


def test_caller_counts_below_zero_become_done():
    """schedule.py:85-94 on counts a caller supplies: a pending block whose count
    a commit drops below 0 is never selected (the reference returns [[0]] here)."""
    g = grid_of(1, 2)
    assert P.schedule_all(g, np.array([0, 0], np.int32)) == [[0]]
    g3 = grid_of(3, 3)
    c = np.zeros(9, np.int32)
    assert P.schedule_all(g3, c) == O.schedule_all(O.Grid.of(12, 12, 4), c)


@settings(max_examples=60, deadline=None)
@given(rows=st.integers(1, 8), cols=st.integers(1, 8), seed=st.integers(0, 2**31 - 1))
def test_schedule_arbitrary_counts_match_restatement(rows, cols, seed):
    """Any int counts (including 0s next to each other, large values and -1s)
    give the reference's batch sequence (oracle restatement of schedule.py)."""
    rng = np.random.default_rng(seed)
    c = rng.integers(-2, 40, size=rows * cols).astype(np.int32)
    c[rng.uniform(size=c.size) < 0.2] = 0
    assert P.schedule_all(grid_of(rows, cols), c) == O.schedule_all(O.Grid.of(rows * 4, cols * 4, 4), c)


def test_schedule_rejects_huge_counts():
    with pytest.raises(Exception):
        P.schedule_all(grid_of(2, 2), np.array([0, 1 << 20, 1, 2], np.int32))


@settings(max_examples=40, deadline=None)
@given(rows=st.integers(1, 9), cols=st.integers(1, 9), seed=st.integers(0, 2**31 - 1),
       density=st.floats(0.05, 1.0))
def test_schedule_properties(rows, cols, seed, density):
    rng = np.random.default_rng(seed)
    table = (rng.uniform(size=(rows, cols)) < density).astype(np.int64)
    g = grid_of(rows, cols)
    counts = P.init_counts(g, table)
    before = counts.copy()
    batches = P.schedule_all(g, counts)
    np.testing.assert_array_equal(counts, before)
    flat = [b for bt in batches for b in bt]
    assert sorted(flat) == np.flatnonzero(table.reshape(-1)).tolist()
    assert all(batches)
    for bt in batches:
        s = set(bt)
        for b in bt:
            assert s.isdisjoint(P.neighbors(g, b))
    lossy = {(r, c) for r in range(rows) for c in range(cols) if table[r, c]}
    assert batches == resimulate(rows, cols, lossy)


def _params(c):
    return P.FseParams(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"],
                       iterations=c["iterations"], block_size=c["block_size"], fft_size=c["fft"])


@pytest.mark.parametrize("i", range(11))
def test_plan_reports_reference_batches(golden, i):
    c = conceal_case(golden("conceal_cases.npz"), i)
    plan = P.build_plan(c["mask"], _params(c), c["order"])
    assert plan.batches() == c["batches"]
    assert plan.unconcealed() == c["unconcealed"]
    assert plan.n_processed == c["processed"]
    # levels are a partition of the processed blocks, never deeper than the batches
    lv = plan.levels()
    assert sorted(b for l in lv for b in l) == sorted(b for bt in c["batches"] for b in bt)
    assert len(lv) <= max(1, len(c["batches"]))


@pytest.mark.parametrize("i", [0, 1, 2, 4, 8, 9, 10])
def test_level_plan_reproduces_reference_on_cpu(golden, i):
    """Rank-based classification + level grouping + racing in-level write-back
    (what the device does) equals the reference's phase-by-phase snapshots."""
    c = conceal_case(golden("conceal_cases.npz"), i)
    plan = P.build_plan(c["mask"], _params(c), c["order"])
    img, msk = emulate_levels(c["image"], c["mask"], c["block_size"], c["d"], c["rho"], c["delta"],
                              c["gamma"], c["iterations"], c["fft"], plan.ranks(), plan.levels(),
                              shuffle_seed=i)
    np.testing.assert_array_equal(msk, c["out_mask"])
    assert np.max(np.abs(img - c["out_image"])) <= 1e-9


def test_full_config_plans_report_reference_batches(golden):
    from paper_2207_00233_b200 import synth
    g = golden("full_cfg.npz")
    for i in range(int(g["n_cases"])):
        img, mask = synth.config_scene(int(g[f"f{i}_config"]))
        assert [int(img.astype(np.int64).sum()), int(mask.astype(np.int64).sum())] == \
            g[f"f{i}_image_sum"].tolist(), "synthetic generator drifted from the golden inputs"
        p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
        plan = P.build_plan(mask, p, str(g[f"f{i}_order"]))
        assert plan.batches() == csr(g[f"f{i}_batch_ptr"], g[f"f{i}_batch_blocks"])


def test_plan_validation_errors():
    m = np.zeros((16, 16), np.uint8)
    with pytest.raises(ValueError):
        P.FseParams(rho=1.0)
    with pytest.raises(ValueError):
        P.FseParams(block_size=0)
    bad = _lib.FseParamsC(-1, 4, 10, 0, 0, 0.8, 0.2, 0.5)
    import ctypes
    h = ctypes.c_void_p()
    rc = _lib.lib().fse_plan_build(m.ctypes.data, 16, 16, ctypes.byref(bad), 0, ctypes.byref(h))
    assert rc == _lib.FSE_EINVAL and b"d must be" in _lib.lib().fse_last_error()


def test_plan_many_threads_equals_single():
    from paper_2207_00233_b200 import synth
    masks = [synth.loss_mask(96, 128, "mixed", 0.3, s) for s in range(6)]
    p = P.FseParams(d=14, iterations=10, block_size=4, fft_size=64)
    many = P.build_plans(masks, p, "optimized", threads=3)
    for m, pl in zip(masks, many):
        one = P.build_plan(m, p)
        assert pl.batches() == one.batches() and pl.levels() == one.levels()
        np.testing.assert_array_equal(pl.ranks(), one.ranks())


def _reference_order(mask, B, d, delta, order):
    """The reference's processing order restated in Python (schedule.py:28-105
    phases or the linescan sequence, conceal.py:145-163 snapshot batches with
    the degeneracy test of fse.py:150-151, conceal.py:69-94 retry sweeps):
    returns (batches, unconcealed)."""
    H, W = mask.shape
    g = O.Grid.of(H, W, B)
    lossy = O.lost_per_block(g, mask).reshape(-1) > 0
    if order == "optimized":
        phases = O.schedule_all(g, O.init_counts(g, lossy.reshape(g.rows, g.cols)))
    else:
        phases = [[b] for b in np.flatnonzero(lossy).tolist()]
    state = mask.copy()

    def usable(b):
        _, cls, _ = O.classify(g, state, b, d)
        return (O.weight_plane(cls.shape, cls, 0.8, delta) > 0).any()

    def write(b):
        r0, r1, c0, c1 = g.bounds(b)
        sub = state[r0:r1, c0:c1]
        sub[sub == O.LOST] = O.RECONSTRUCTED

    batches, deferred = [], []
    for ph in phases:
        ok = [b for b in ph if usable(b)]
        deferred += [b for b in ph if b not in ok]
        for b in ok:  # snapshot: writes land after the whole batch
            write(b)
        if ok:
            batches.append(ok)
    pending = sorted(deferred)
    for _ in range(max(g.rows, g.cols)):
        if not pending:
            break
        still = []
        for b in pending:
            if usable(b):
                write(b)
                batches.append([b])
            else:
                still.append(b)
        if len(still) == len(pending):
            break
        pending = still
    return batches, pending


def test_plan_matches_python_restatement_on_random_masks():
    """build_plan (C++: bucket-queue scheduler, static/dynamic usability,
    retry sweeps, dependency levels) against the Python restatement of the
    reference's order on random masks: ragged grids, RECONSTRUCTED samples,
    delta = 0 (R samples weightless), fully lost frames, both orders.  Levels
    must order every pair of overlapping blocks like their ranks."""
    rng = np.random.default_rng(17)
    for t in range(120):
        H, W = int(rng.integers(1, 48)), int(rng.integers(1, 48))
        B, d = int(rng.integers(1, 7)), int(rng.integers(0, 12))
        delta = float(rng.choice([0.0, 0.2]))
        order = str(rng.choice(["optimized", "linescan"]))
        mask = rng.choice(np.array([0, 1, 2], dtype=np.uint8), size=(H, W), p=rng.dirichlet([1, 1, 0.3]))
        if t % 10 == 0:
            mask[:] = 1
        mask = np.ascontiguousarray(mask)
        p = P.FseParams(d=d, delta=delta, iterations=5, block_size=B)
        plan = P.build_plan(mask, p, order)
        batches, unconcealed = _reference_order(mask, B, d, delta, order)
        assert plan.batches() == batches, (t, H, W, B, d, delta, order)
        assert plan.unconcealed() == unconcealed
        # levels: a block's level exceeds that of every lower-rank block its window covers
        rk = plan.ranks()
        lv = np.full(rk.shape, -1)
        for l, blocks in enumerate(plan.levels()):
            lv[blocks] = l
        R = -(-d // B) if d > 0 else 0
        cols = plan.cols
        for b in np.flatnonzero(lv >= 0):
            r, c = divmod(int(b), cols)
            for rr in range(max(0, r - R), min(plan.rows, r + R + 1)):
                for cc in range(max(0, c - R), min(cols, c + R + 1)):
                    o = rr * cols + cc
                    if lv[o] >= 0 and rk[o] < rk[b]:
                        assert lv[o] < lv[b]


def test_abi_argument_errors_without_a_device():
    """Entry points added for the fused halo exchange and the level-width
    switch reject bad arguments with the ABI's error codes before touching
    CUDA (no exception crosses the C boundary)."""
    import ctypes

    L = _lib.lib()
    assert L.fse_shard_set_peers(None, None, None, None, None, None, 1) == _lib.FSE_EINVAL
    assert L.fse_ipc_handle(None, None) == _lib.FSE_EINVAL
    assert L.fse_ipc_open(None, None) == _lib.FSE_EINVAL
    assert L.fse_ipc_close(ctypes.c_void_p(0x1234)) == _lib.FSE_EINVAL
    assert L.fse_flags_alloc(None) == _lib.FSE_EINVAL
    assert L.fse_set_track_below(-1) == _lib.FSE_EINVAL
    assert b"track_below" in L.fse_last_error()
    assert L.fse_shard_run(None, 0, 1, None) == _lib.FSE_EINVAL


@pytest.mark.parametrize("name", ["cfg3", "cfg4f0", "cfg5crop", "cfg3def"])
def test_large_golden_batches_from_cpp_planner(golden, name):
    """The C++ planner's batches on full-size frames equal the reference's
    (tests/golden/make_golden_large.py), and the fixture's sampled full pick
    sequences agree with its per-block hashes."""
    from helpers import large_case, pick_hash

    g = golden(f"large_{name}.npz")
    img, mask, kw, fft = large_case(g)
    plan = P.build_plan(mask, P.FseParams(fft_size=fft, **kw))
    assert plan.batches() == csr(g["batch_ptr"], g["batch_blocks"])
    assert plan.unconcealed() == g["unconcealed"].tolist()
    idx = np.searchsorted(g["pick_blocks"], g["sample_blocks"])
    np.testing.assert_array_equal(pick_hash(g["sample_picks"]), g["pick_hash"][idx])


def _plan_sig(pl):
    return pl.batches(), pl.levels(), pl.ranks().tolist(), pl.unconcealed(), pl.n_levels


def test_band_parallel_planner_equals_sequential_on_random_masks():
    """fse_plan_build_threads: the band-parallel planner (per-phase minimum,
    first-row fix-up, band-local commits, rank + level pass fused) gives the
    sequential planner's plan for every thread count -- down to bands of one
    block row, where fix-ups reach the band's last row and the ordered redo
    path runs."""
    rng = np.random.default_rng(7)
    checked = 0
    for trial in range(60):
        H, W = int(rng.integers(8, 100)), int(rng.integers(8, 100))
        B = int(rng.choice([2, 3, 4, 8]))
        d = int(rng.choice([0, 2, 5, 14]))
        kind = trial % 4
        if kind == 0:
            mask = (rng.random((H, W)) < rng.uniform(0.05, 0.9)).astype(np.uint8)
        elif kind == 1:
            bm = rng.random(((H + B - 1) // B, (W + B - 1) // B)) < rng.uniform(0.1, 0.95)
            mask = np.kron(bm, np.ones((B, B), np.uint8))[:H, :W].astype(np.uint8)
        elif kind == 2:
            mask = np.ones((H, W), np.uint8)
            mask[rng.random((H, W)) < 0.02] = 0
        else:
            mask = (rng.random((H, W)) < 0.5).astype(np.uint8)
            mask[rng.random((H, W)) < 0.1] = 2
        p = P.FseParams(d=d, iterations=10, block_size=B, delta=float(rng.choice([0.0, 0.2])))
        ref = _plan_sig(P.build_plan(mask, p, plan_threads=1))
        rows = (H + B - 1) // B
        for T in sorted({2, 3, 5, rows}):
            if T <= rows:
                assert _plan_sig(P.build_plan(mask, p, plan_threads=T)) == ref, (trial, T)
                checked += 1
    assert checked > 150


@pytest.mark.parametrize("name", ["cfg3", "cfg5crop"])
def test_large_golden_batches_for_every_plan_thread_count(golden, name):
    from helpers import large_case

    g = golden(f"large_{name}.npz")
    img, mask, kw, fft = large_case(g)
    p = P.FseParams(fft_size=fft, **kw)
    want = csr(g["batch_ptr"], g["batch_blocks"])
    ref = None
    for T in (1, 3, 8, 16):
        pl = P.build_plan(mask, p, plan_threads=T)
        assert pl.batches() == want, T
        sig = _plan_sig(pl)
        ref = ref or sig
        assert sig == ref, T


def test_plan_export_import_round_trip_and_rejects_corrupt_bytes():
    """fse_plan_export / fse_plan_import (one rank plans, the others import):
    the imported plan is the plan; truncated or foreign bytes are rejected."""
    from paper_2207_00233_b200 import synth

    _, mask = synth.config_scene(3)
    p = P.FseParams(d=14, iterations=10, block_size=4, fft_size=64)
    a = P.build_plan(mask, p)
    data = a.to_bytes()
    b = P.Plan.from_bytes(data)
    assert _plan_sig(a) == _plan_sig(b)
    assert (a.rows, a.cols, a.n_lossy, a.max_wr, a.max_wc) == (b.rows, b.cols, b.n_lossy, b.max_wr, b.max_wc)
    with pytest.raises(ValueError, match="truncated"):
        P.Plan.from_bytes(data[: len(data) // 2])
    with pytest.raises(ValueError, match="not a serialised plan"):
        P.Plan.from_bytes(b"\0" * len(data))


@pytest.mark.parametrize("shape,B,fill", [((1, 200), 1, 1.0), ((300, 1), 1, 0.7), ((64, 64), 4, 1.0),
                                          ((64, 64), 4, 0.0), ((96, 40), 2, 0.97), ((17, 300), 3, 0.5)])
def test_band_parallel_planner_edge_grids(shape, B, fill):
    """Degenerate grids for the band-parallel planner: one block row or column,
    everything lost (every window degenerate: all blocks unconcealed), nothing
    lost, almost everything lost -- identical to the sequential planner for
    every thread count."""
    rng = np.random.default_rng(int(fill * 100) + shape[0])
    mask = (rng.random(shape) < fill).astype(np.uint8)
    for delta in (0.0, 0.2):
        p = P.FseParams(d=5, iterations=5, block_size=B, delta=delta)
        ref = _plan_sig(P.build_plan(mask, p, plan_threads=1))
        rows = -(-shape[0] // B)
        for T in (2, 3, 7, rows):
            assert _plan_sig(P.build_plan(mask, p, plan_threads=T)) == ref, (T, delta)


# ---- level balancing (fse_plan_rebalance): a pure re-leveling

def _check_balanced(plan, lv0, ranks0, batches0, params):
    lv1 = plan.levels()
    assert sorted(b for l in lv0 for b in l) == sorted(b for l in lv1 for b in l)
    assert len(lv1) == len(lv0)
    np.testing.assert_array_equal(plan.ranks(), ranks0)  # ranks and batches untouched
    assert plan.batches() == batches0
    rows, cols = plan.rows, plan.cols
    level = np.full(rows * cols, -1)
    for l, bl in enumerate(lv1):
        level[bl] = l
    R = -(-params.d // params.block_size)
    L2, R2 = level.reshape(rows, cols), ranks0.reshape(rows, cols)
    for r, c in np.argwhere(L2 >= 0):
        r0, r1, c0, c1 = max(0, r - R), min(rows, r + R + 1), max(0, c - R), min(cols, c + R + 1)
        dep = (R2[r0:r1, c0:c1] < R2[r, c]) & (L2[r0:r1, c0:c1] >= 0)
        # every lower-rank block whose samples the window covers runs in an earlier launch
        assert not dep.any() or L2[r0:r1, c0:c1][dep].max() < L2[r, c], (r, c)
    return lv1


@pytest.mark.parametrize("narrow,wave", [(3, 0), (8, 0), (4, 12), (1, 0)])
def test_rebalance_keeps_ranks_and_true_dependences(narrow, wave):
    rng = np.random.default_rng(narrow * 100 + wave)
    for shape, B, d in [((96, 128), 4, 14), ((70, 90), 8, 9), ((64, 64), 2, 5)]:
        mask = (rng.uniform(size=(shape[0] // 8 + 1, shape[1] // 8 + 1)) < 0.45).astype(np.uint8)
        mask = np.kron(mask, np.ones((8, 8), np.uint8))[:shape[0], :shape[1]]
        p = P.FseParams(d=d, iterations=5, block_size=B, fft_size=64)
        for order in ("optimized", "linescan"):
            plan = P.build_plan(mask, p, order)
            lv0, ranks0, batches0 = plan.levels(), plan.ranks(), plan.batches()
            moved = plan.rebalance(narrow, wave)
            lv1 = _check_balanced(plan, lv0, ranks0, batches0, p)
            assert (moved > 0) == (lv1 != lv0)
            if wave == 0:  # no level that accepted blocks grew past `narrow`
                for a, b in zip(lv0, lv1):
                    assert len(b) <= max(len(a), narrow)
            # narrow = 0 is a no-op; a second pass finds nothing worse
            assert plan.rebalance(0, 0) == 0
            _check_balanced(plan, lv1, ranks0, batches0, p)


@pytest.mark.parametrize("i", [0, 1, 2, 4, 8, 9, 10])
def test_balanced_level_plan_reproduces_reference_on_cpu(golden, i):
    """The device pipeline emulated on the CPU over BALANCED levels (blocks with
    slack moved into later, narrower levels) still equals the reference's
    phase-by-phase result (conceal.py:97-181): only true dependences matter."""
    c = conceal_case(golden("conceal_cases.npz"), i)
    plan = P.build_plan(c["mask"], _params(c), c["order"])
    lv0 = plan.levels()
    plan.rebalance(2, 0)
    img, msk = emulate_levels(c["image"], c["mask"], c["block_size"], c["d"], c["rho"], c["delta"],
                              c["gamma"], c["iterations"], c["fft"], plan.ranks(), plan.levels(),
                              shuffle_seed=i)
    np.testing.assert_array_equal(msk, c["out_mask"])
    assert np.max(np.abs(img - c["out_image"])) <= 1e-9
    assert sorted(b for l in lv0 for b in l) == sorted(b for l in plan.levels() for b in l)


def test_rebalance_survives_export_import_and_rejects_bad_arguments():
    rng = np.random.default_rng(5)
    mask = np.kron((rng.uniform(size=(10, 12)) < 0.5).astype(np.uint8), np.ones((8, 8), np.uint8))
    p = P.FseParams(d=14, iterations=3, block_size=4, fft_size=64)
    plan = P.build_plan(mask, p)
    plan.rebalance(5, 0)
    twin = P.Plan.from_bytes(plan.to_bytes())
    assert twin.levels() == plan.levels()
    L = _lib.lib()
    assert L.fse_plan_rebalance(plan.handle, -1, 0, None) == _lib.FSE_EINVAL
    assert L.fse_plan_rebalance(None, 1, 0, None) == _lib.FSE_EINVAL
