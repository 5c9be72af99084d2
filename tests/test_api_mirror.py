"""The reference's host-side API tests for the concealment path, restated
against this package (CPU; no kernel calls).

Each test names the reference test it mirrors (fsefill tests/test_grid.py,
test_schedule.py, test_fse.py).  Expected values come from the algorithm's
definition (brute force or the oracle restatement in oracle/oracle.py), so a
user of the reference switching to this package keeps the same behaviour:
same names, argument meanings, return shapes and exceptions.
"""

import numpy as np
import pytest

import paper_2207_00233_b200 as P
from oracle import oracle as O


# ------------------------------------------------------------------ grid.py
def test_build_grid_rounds_up():  # test_grid.py: test_build_grid_rounds_up
    g = P.build_grid(33, 17, 16)  # (width, height) as in the reference
    assert (g.rows, g.cols, g.n_blocks) == (2, 3, 6)
    with pytest.raises(ValueError):
        P.build_grid(0, 5, 4)
    with pytest.raises(ValueError):
        P.build_grid(5, 5, 0)


def test_block_index_round_trip_and_bounds():  # test_block_rc_index_round_trip / _bounds_clip
    g = P.build_grid(33, 17, 16)
    for b in range(g.n_blocks):
        assert g.block_index(*g.block_rc(b)) == b
    for bad in (-1, g.n_blocks):
        with pytest.raises(IndexError):
            g.block_rc(bad)
    # ragged right column (1 sample wide) and bottom row (1 sample tall)
    assert g.block_bounds(0) == (0, 16, 0, 16)
    assert g.block_bounds(2) == (0, 16, 32, 33)
    assert g.block_bounds(5) == (16, 17, 32, 33)


def test_edges_touched_and_neighbors():  # test_edges_touched / test_neighbors_*
    g = P.build_grid(48, 48, 16)
    assert [g.edges_touched(g.block_index(r, c)) for r, c in ((0, 0), (0, 1), (1, 1))] == [2, 1, 0]
    assert P.build_grid(8, 8, 16).edges_touched(0) == 4
    for b in range(g.n_blocks):  # row-major 8-neighbourhood, brute force
        r, c = g.block_rc(b)
        want = [rr * g.cols + cc for rr in range(g.rows) for cc in range(g.cols)
                if max(abs(rr - r), abs(cc - c)) == 1]
        assert P.neighbors(g, b) == want
    assert P.neighbors(P.build_grid(4, 4, 16), 0) == []


def test_classify_window_clips_and_labels():  # test_classify_window_clips_and_labels
    g = P.build_grid(32, 32, 8)
    mask = np.full((32, 32), P.KNOWN, dtype=np.uint8)
    mask[8:16, 8:16] = P.LOST          # the block itself
    mask[4:6, 10:12] = P.LOST          # a loss outside the block
    mask[20:24, 4:8] = P.RECONSTRUCTED
    win = P.classify_window(g, mask, g.block_index(1, 1), d=16)
    assert win.origin == (0, 0) and win.shape == (32, 32) and win.block_rect == (8, 16, 8, 16)
    cls = win.cls
    assert (cls[8:16, 8:16] == P.AREA_BI).all()
    assert (cls[4:6, 10:12] == P.AREA_BO).all()
    assert (cls[20:24, 4:8] == P.AREA_R).all()
    counts = {int(v): int((cls == v).sum()) for v in (P.AREA_A, P.AREA_BI, P.AREA_BO, P.AREA_R)}
    assert counts == {int(P.AREA_BI): 64, int(P.AREA_BO): 4, int(P.AREA_R): 16,
                      int(P.AREA_A): 32 * 32 - 84}


def test_classify_window_interior_and_shape_check():  # _interior_not_clipped / _rejects_shape_mismatch
    g = P.build_grid(64, 64, 8)
    win = P.classify_window(g, np.full((64, 64), P.KNOWN, dtype=np.uint8), g.block_index(3, 3), d=4)
    assert (win.origin, win.shape, win.block_rect) == ((20, 20), (16, 16), (4, 12, 4, 12))
    assert (win.cls == P.AREA_A).all()
    with pytest.raises(ValueError):
        P.classify_window(P.build_grid(32, 32, 8), np.zeros((16, 16), dtype=np.uint8), 0, 4)


def test_classify_window_matches_oracle_on_random_masks():
    rng = np.random.default_rng(11)
    for _ in range(20):
        H, W, B, d = int(rng.integers(5, 40)), int(rng.integers(5, 40)), int(rng.integers(1, 9)), int(rng.integers(0, 9))
        mask = rng.choice([P.KNOWN, P.LOST, P.RECONSTRUCTED], size=(H, W), p=[0.6, 0.3, 0.1]).astype(np.uint8)
        g, og = P.build_grid(W, H, B), O.Grid.of(H, W, B)
        for b in rng.integers(0, g.n_blocks, size=5).tolist():
            win = P.classify_window(g, mask, b, d)
            want = O.classify(og, mask, b, d)
            assert win.origin == want[0]
            np.testing.assert_array_equal(win.cls, want[1])
            assert win.block_rect == want[2]


def test_lost_per_block_matches_brute_force():  # test_lost_per_block_matches_brute_force
    rng = np.random.default_rng(3)
    mask = np.where(rng.uniform(size=(37, 53)) < 0.3, P.LOST, P.KNOWN).astype(np.uint8)
    g = P.build_grid(53, 37, 8)
    table = P.lost_per_block(g, mask)
    assert table.shape == (g.rows, g.cols)
    for b in range(g.n_blocks):
        r0, r1, c0, c1 = g.block_bounds(b)
        assert table[g.block_rc(b)] == int((mask[r0:r1, c0:c1] == P.LOST).sum())


# -------------------------------------------------------------- schedule.py
def _lossy(rows, cols, on):
    t = np.zeros((rows, cols), dtype=np.int64)
    for r, c in on:
        t[r, c] = 1
    return t


def test_init_counts_bonuses():  # test_single_block_grid_* / _isolated_interior_* / _margin_and_corner_*
    one = P.build_grid(4, 4, 16)
    counts = P.init_counts(one, np.ones((1, 1)))
    assert counts.tolist() == [5] and P.schedule_all(one, counts) == [[0]]
    g = P.build_grid(5 * 16, 5 * 16, 16)
    counts = P.init_counts(g, _lossy(5, 5, [(2, 2)]))
    assert counts[g.block_index(2, 2)] == 0
    assert all(c == -1 for i, c in enumerate(counts.tolist()) if i != g.block_index(2, 2))
    g3 = P.build_grid(48, 48, 16)
    assert P.init_counts(g3, np.ones((3, 3))).tolist() == [8] * 9  # corners 3+5, edges 5+3, centre 8


def test_init_counts_matches_oracle_on_random_grids():
    rng = np.random.default_rng(5)
    for _ in range(50):
        rows, cols = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        table = (rng.uniform(size=(rows, cols)) < rng.uniform(0.1, 0.9)).astype(np.int64)
        g = P.build_grid(cols * 4, rows * 4, 4)
        np.testing.assert_array_equal(P.init_counts(g, table),
                                      O.init_counts(O.Grid.of(rows * 4, cols * 4, 4), table))


def test_all_lossy_3x3_batch_sequence_and_commit():  # _all_lossy_3x3_* / _commit_batch_releases_*
    g = P.build_grid(48, 48, 16)
    counts = P.init_counts(g, np.ones((3, 3)))
    assert P.select_batch(g, counts) == [0, 2, 6, 8]  # corners first, row-major, non-adjacent
    assert P.schedule_all(g, counts) == [[0, 2, 6, 8], [4], [1, 7], [3, 5]]
    c = counts.copy()
    P.commit_batch(g, c, [0, 2, 6, 8])
    want = counts.copy()
    for b in (0, 2, 6, 8):  # members to -1, each neighbour decremented once per member
        want[b] = -1
    for b in (0, 2, 6, 8):
        for nb in P.neighbors(g, b):
            want[nb] -= 1
    np.testing.assert_array_equal(c, want)
    assert c.tolist() == [-1, 6, -1, 6, 4, 6, -1, 6, -1]
    P.commit_batch(g, c, [4])  # drift below -1 is allowed
    assert c.tolist() == [-2, 5, -2, 5, -1, 5, -2, 5, -2]


def test_select_batch_empty_and_no_loss():  # _select_batch_empty_raises / _no_loss_schedules_nothing
    g = P.build_grid(48, 48, 16)
    counts = P.init_counts(g, np.zeros((3, 3)))
    assert (counts == -1).all() and P.schedule_all(g, counts) == []
    with pytest.raises(P.EmptyScheduleError):
        P.select_batch(g, counts)


def test_schedule_all_does_not_mutate_and_matches_select_commit():  # _does_not_mutate_input
    rng = np.random.default_rng(7)
    for _ in range(30):
        rows, cols = int(rng.integers(1, 10)), int(rng.integers(1, 10))
        g = P.build_grid(cols * 8, rows * 8, 8)
        counts = P.init_counts(g, (rng.uniform(size=(rows, cols)) < 0.5).astype(np.int64))
        before = counts.copy()
        got = P.schedule_all(g, counts)
        np.testing.assert_array_equal(counts, before)
        c, want = counts.copy(), []  # the single-step rules, applied until nothing is pending
        while (c >= 0).any():
            batch = P.select_batch(g, c)
            P.commit_batch(g, c, batch)
            want.append(batch)
        assert got == want


def test_render_batch_trace():  # test_render_batch_trace_format / _marks_unscheduled
    g = P.build_grid(48, 48, 16)
    assert P.render_batch_trace(g, [[0, 2, 6, 8], [4], [1, 7], [3, 5]]) == "1 3 1\n4 2 4\n1 3 1"
    assert P.render_batch_trace(P.build_grid(32, 32, 16), [[0]]) == "1 -1\n-1 -1"


# ------------------------------------------------------------------- fse.py
@pytest.mark.parametrize("kwargs", [{"d": -1}, {"rho": 0.0}, {"rho": 1.0}, {"delta": -0.1},
                                    {"delta": 1.5}, {"gamma": 0.0}, {"gamma": 1.2},
                                    {"iterations": -1}, {"block_size": 0}, {"fft_size": 0}])
def test_params_validation(kwargs):  # test_fse.py: test_params_validation
    with pytest.raises(ValueError):
        P.FseParams(**kwargs)


def test_params_defaults():  # test_fse.py: test_params_defaults
    p = P.FseParams()
    assert (p.d, p.rho, p.delta, p.gamma, p.iterations, p.block_size, p.fft_size) == (
        16, 0.8, 0.2, 0.5, 200, 16, None)


def test_weight_plane_centre_classes_and_scalar_twin():  # _weight_center_and_classes / _matches_scalar
    p = P.FseParams(rho=0.7, delta=0.3)
    rng = np.random.default_rng(1)
    for shape in ((9, 9), (8, 6), (1, 5)):  # even sizes: centre between samples
        cls = rng.integers(0, 4, size=shape).astype(np.uint8)
        w = P.weight_plane(shape, cls, p)
        for m in range(shape[0]):
            for n in range(shape[1]):
                # vectorised and scalar pow may differ in the last ulp (as in the reference)
                assert w[m, n] == pytest.approx(P.weight(m, n, shape, int(cls[m, n]), p), rel=1e-12)
        assert (w[(cls == P.AREA_BI) | (cls == P.AREA_BO)] == 0).all()
        np.testing.assert_array_equal(w, O.weight_plane(shape, cls, p.rho, p.delta))
    w = P.weight_plane((9, 9), np.zeros((9, 9), dtype=np.uint8), p)
    assert w[4, 4] == 1.0 and w.max() == 1.0


def test_dft_basis_unit_modulus_and_orthogonality():  # test_fse.py: same name
    shape = (6, 5)
    basis = np.stack([P.dft_basis(shape, (k1, k2)).reshape(-1) for k1 in range(6) for k2 in range(5)])
    np.testing.assert_allclose(np.abs(basis), 1.0, atol=1e-12)
    np.testing.assert_allclose(basis @ basis.conj().T, 30.0 * np.eye(30), atol=1e-9)


def test_degenerate_window_raises_before_any_device_work():  # test_degenerate_window_raises
    cls = np.full((8, 8), P.AREA_BI, dtype=np.uint8)
    win = P.Window(origin=(0, 0), cls=cls, block_rect=(0, 8, 0, 8), values=np.zeros((8, 8)))
    with pytest.raises(P.DegenerateWindowError):
        P.generate_model(win, P.FseParams(iterations=5))
    assert issubclass(P.DegenerateWindowError, ValueError)


def test_backend_registry():  # test_set_backend_round_trip
    name = P.get_backend()
    P.set_backend(name)
    assert P.get_backend() == name
    with pytest.raises(ValueError):
        P.set_backend("fortran")


def test_conceal_argument_errors_without_device_work():  # conceal.py:113-120
    img = np.zeros((16, 16))
    msk = np.zeros((16, 16), dtype=np.uint8)
    with pytest.raises(ValueError):
        P.conceal(img, msk, order="zigzag")
    with pytest.raises(ValueError):
        P.conceal(img, msk, threads=0)
    with pytest.raises(ValueError):
        P.conceal(img, msk, order="linescan", threads=2)
    with pytest.raises(ValueError):
        P.conceal(img, np.zeros((8, 16), dtype=np.uint8))


def test_stream_needs_a_device():
    """No CPU fallback: the streaming API refuses to run without CUDA."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError):
        P.ConcealStream(P.FseParams(), (16, 16))
