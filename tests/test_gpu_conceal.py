"""End-to-end concealment on the GPU (conceal / conceal_batch through
fse_conceal_frames) against the reference's golden outputs, plus the
reference's pipeline properties (test_conceal.py, test_acceptance.py)."""

import os

import numpy as np
import pytest

from helpers import conceal_case, csr
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2207_00233_b200")
from paper_2207_00233_b200 import synth  # noqa: E402


def _params(c):
    return P.FseParams(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"],
                       iterations=c["iterations"], block_size=c["block_size"], fft_size=c["fft"])


def psnr(orig, res, mask):
    region = mask != 0
    mse = float(np.mean((orig[region] - res[region]) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(255.0 ** 2 / mse)


@pytest.mark.parametrize("i", range(11))
def test_fp64_matches_reference_golden(golden, i):
    c = conceal_case(golden("conceal_cases.npz"), i)
    img, msk, rep, picks = P.conceal(c["image"], c["mask"], _params(c), c["order"],
                                     precision="fp64", return_picks=True)
    np.testing.assert_array_equal(msk, c["out_mask"])
    assert rep.batches == c["batches"]
    assert rep.unconcealed_blocks == c["unconcealed"]
    assert rep.blocks_processed == c["processed"]
    assert np.max(np.abs(img - c["out_image"])) <= 1e-6
    if c["fft"] is not None:
        for b, want in zip(c["pick_blocks"].tolist(), c["picks"]):
            assert O.canonical_picks(picks[b], c["fft"]) == [tuple(x) for x in want.tolist()], b


# fp32 tolerance.  Greedy basis selection is chaotic on these
# windows: a near-tie the fp64 reference separates by ~1e-6 relative (golden
# case 2, block 94, iteration 59) or an ill-conditioned window that amplifies
# rounding (tools/fp32_stats.py) switches one pick, and the switched block then
# feeds later blocks as reconstructed samples.  fp32 rounding moves |g|^2 by up
# to ~1e-4 of the running maximum, so no fp32 kernel reproduces the fp64 picks
# everywhere; the per-sample 0.5 bound holds where no switch happens (cases 6
# and 7) and image PSNR stays within FP32_PSNR_DB of the reference elsewhere.
# Exact parity is the fp64 path's job (test_fp64_matches_reference_golden).
FP32_PSNR_DB = 0.15


@pytest.mark.parametrize("i", [6, 7])
def test_fp32_within_half_grey_level_when_picks_agree(golden, i):
    c = conceal_case(golden("conceal_cases.npz"), i)
    img, msk, _ = P.conceal(c["image"], c["mask"], _params(c), c["order"], precision="fp32")
    np.testing.assert_array_equal(msk, c["out_mask"])
    assert np.max(np.abs(img - c["out_image"])) <= 0.5


@pytest.mark.parametrize("i", [2, 3, 4, 5, 6, 7])
def test_fp32_psnr_parity_with_reference(golden, i):
    c = conceal_case(golden("conceal_cases.npz"), i)
    img, msk, _ = P.conceal(c["image"], c["mask"], _params(c), c["order"], precision="fp32")
    np.testing.assert_array_equal(msk, c["out_mask"])
    truth = c["image"].astype(np.float64)
    assert abs(psnr(truth, img, c["mask"]) - psnr(truth, c["out_image"], c["mask"])) <= FP32_PSNR_DB
    assert np.isfinite(img).all()


@pytest.mark.parametrize("k", [0, 1, 2])
def test_full_baseline_configs_fp64_identical_picks(golden, k):
    """BASELINE configs 1 and 2 at full size, fp64: every block's canonical pick
    sequence identical to the reference, every sample within 1e-6."""
    g = golden("full_cfg.npz")
    img, mask = synth.config_scene(int(g[f"f{k}_config"]))
    p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
    out, msk, rep, picks = P.conceal(img, mask, p, str(g[f"f{k}_order"]), precision="fp64",
                                     return_picks=True)
    assert rep.batches == csr(g[f"f{k}_batch_ptr"], g[f"f{k}_batch_blocks"])
    lost = mask == 1
    assert np.max(np.abs(out[lost] - g[f"f{k}_lost_values"])) <= 1e-6
    assert int(msk.astype(np.int64).sum()) == int(g[f"f{k}_out_mask_sum"])
    bad = [b for b, want in zip(g[f"f{k}_pick_blocks"].tolist(), g[f"f{k}_picks"])
           if O.canonical_picks(picks[b], (64, 64)) != [tuple(x) for x in want.astype(int).tolist()]]
    assert bad == []


@pytest.mark.parametrize("k", [0, 1])
def test_full_baseline_configs_fp32_tolerance(golden, k):
    g = golden("full_cfg.npz")
    img, mask = synth.config_scene(int(g[f"f{k}_config"]))
    p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
    out, _, _ = P.conceal(img, mask, p, str(g[f"f{k}_order"]), precision="fp32")
    lost = mask == 1
    ref = img.astype(np.float64).copy()
    ref[lost] = g[f"f{k}_lost_values"]
    truth = img.astype(np.float64)
    assert abs(psnr(truth, out, mask) - psnr(truth, ref, mask)) <= FP32_PSNR_DB
    # most samples are unaffected by pick switches
    assert np.mean(np.abs(out[lost] - ref[lost]) <= 0.5) >= 0.6


def scene(shape=(64, 64)):
    y, x = np.mgrid[0:shape[0], 0:shape[1]].astype(np.float64)
    return 120.0 + 50.0 * np.sin(x / 5.0) + 30.0 * np.cos(y / 7.0) + 0.3 * x


FAST = None


def fast():
    return P.FseParams(d=8, iterations=30, block_size=8)


def square_loss(shape, squares):
    m = np.zeros(shape, np.uint8)
    for r, c, s in squares:
        m[r:r + s, c:c + s] = 1
    return m


def test_no_loss_is_a_no_op():
    img = scene()
    mask = np.zeros(img.shape, np.uint8)
    for order in ("linescan", "optimized"):
        out, om, rep = P.conceal(img, mask, fast(), order)
        np.testing.assert_array_equal(out, img)
        np.testing.assert_array_equal(om, mask)
        assert rep.blocks_processed == 0 and rep.batches == [] and rep.unconcealed_blocks == []


def test_inputs_not_modified_and_known_preserved():
    img = scene()
    mask = square_loss(img.shape, [(8, 8, 12), (30, 40, 10), (50, 2, 6)])
    i0, m0 = img.copy(), mask.copy()
    for order in ("linescan", "optimized"):
        out, om, rep = P.conceal(img, mask, fast(), order)
        np.testing.assert_array_equal(img, i0)
        np.testing.assert_array_equal(mask, m0)
        known = mask == 0
        np.testing.assert_array_equal(out[known], img[known])
        assert not (om == 1).any() and (om[mask == 1] == 2).all() and (om[known] == 0).all()
        assert rep.order == order and rep.wall_time >= 0


def test_partially_lost_block_keeps_known_half():
    img = scene()
    mask = np.zeros(img.shape, np.uint8)
    mask[16:20, 16:24] = 1
    out, om, _ = P.conceal(img, mask, fast())
    np.testing.assert_array_equal(out[20:24, 16:24], img[20:24, 16:24])
    assert (om[16:20, 16:24] == 2).all() and (om[20:24, 16:24] == 0).all()


def test_argument_errors():
    img = scene()
    mask = square_loss(img.shape, [(8, 8, 8)])
    with pytest.raises(ValueError, match="sequential"):
        P.conceal(img, mask, fast(), order="linescan", threads=2)
    with pytest.raises(ValueError, match="order"):
        P.conceal(img, mask, fast(), order="zigzag")
    with pytest.raises(ValueError, match="threads"):
        P.conceal(img, mask, fast(), threads=0)
    with pytest.raises(ValueError, match="shape"):
        P.conceal(img, mask[:32, :32], fast())
    with pytest.raises(ValueError):
        P.conceal(img, mask, P.FseParams(d=14, block_size=4, iterations=5, fft_size=16))


@pytest.mark.parametrize("threads", [2, 8])
def test_thread_count_invariance(threads):
    img = scene()
    mask = square_loss(img.shape, [(4, 4, 10), (24, 24, 16), (40, 8, 8), (8, 44, 12)])
    a = P.conceal(img, mask, fast(), threads=1)
    b = P.conceal(img, mask, fast(), threads=threads)
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    assert b[2].threads == threads


def test_all_lost_and_retry_sweeps():
    img = scene((32, 32))
    out, om, rep = P.conceal(img, np.ones((32, 32), np.uint8), fast())
    assert (om == 1).all() and rep.blocks_processed == 0
    np.testing.assert_array_equal(out, img)
    assert rep.unconcealed_blocks == list(range(16))
    img = scene((96, 96))
    mask = square_loss(img.shape, [(16, 16, 64)])
    out, om, rep = P.conceal(img, mask, P.FseParams(d=4, iterations=20, block_size=8))
    assert not (om == 1).any() and rep.blocks_processed == 64 and rep.unconcealed_blocks == []
    seen = [b for bt in rep.batches for b in bt]
    assert len(seen) == len(set(seen)) == 64


@pytest.mark.parametrize("nf", [3, 9, 17])
def test_conceal_batch_equals_per_frame(nf):
    """One-chunk batches (< 4 frames) and the staged pipeline (first chunk, the
    rest uploaded and downloaded on the copy stream; a third, small chunk from
    16 frames on) equal per-frame conceal."""
    import torch

    frames = [synth.synthetic_frame(96, 160, 50 + f, 6, 3) for f in range(nf)]
    masks = [synth.loss_mask(96, 160, "mixed", 0.25, 60 + f) for f in range(nf)]
    p = P.FseParams(d=14, iterations=40, block_size=4, fft_size=64)
    for prec in ("fp64", "fp32"):
        if nf > 3:  # pinned uint8 inputs and reused pinned outputs, as bench.py's e2e
            ih = torch.from_numpy(np.stack(frames).astype(np.uint8)).pin_memory()
            frames = [f.astype(np.uint8) for f in frames]
            mh = torch.from_numpy(np.stack(masks)).pin_memory()
            tdt = torch.float64 if prec == "fp64" else torch.float32
            oi = torch.empty(ih.shape, dtype=tdt, pin_memory=True)
            om_ = torch.empty(mh.shape, dtype=torch.uint8, pin_memory=True)
            imgs, msks, reps = P.conceal_batch(ih, mh, p, precision=prec, out_images=oi, out_masks=om_)
        else:
            imgs, msks, reps = P.conceal_batch(np.stack(frames), np.stack(masks), p, precision=prec)
        for f in range(nf):
            one, om, rep = P.conceal(frames[f], masks[f], p, precision=prec)
            assert imgs[f].astype(np.float64).tobytes() == one.tobytes()
            np.testing.assert_array_equal(msks[f], om)
            assert reps[f].batches == rep.batches


def test_deterministic_repeat():
    img, mask = synth.config_scene(2)
    p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
    a = P.conceal(img, mask, p, precision="fp32")[0]
    b = P.conceal(img, mask, p, precision="fp32")[0]
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("B,F", [(2, 32), (4, 64), (8, 128)])
def test_config5_block_sizes_on_a_crop_vs_oracle(B, F):
    img, mask = synth.config_scene(5)
    img, mask = img[:96, :128].copy(), mask[:96, :128].copy()
    p = P.FseParams(d=14, iterations=30, block_size=B, fft_size=F)
    out, om, rep = P.conceal(img, mask, p, precision="fp64")
    o_img, o_msk, o_rep = O.conceal(img, mask, O.Params(d=14, iterations=30, block_size=B, fft_size=(F, F)),
                                    "optimized", kernel="auto")
    assert rep.batches == o_rep.batches
    np.testing.assert_array_equal(om, o_msk)
    assert np.max(np.abs(out - o_img)) <= 1e-6


@pytest.mark.parametrize("config,prec,iters", [(3, "fp32", 200), (4, "fp32", 100)])
def test_full_size_properties(config, prec, iters):
    """BASELINE configs 3 and 4 at full 1080p size: size-independent properties."""
    img, mask = synth.config_scene(config)
    p = P.FseParams(d=14, iterations=iters, block_size=4, fft_size=64)
    out, om, rep = P.conceal(img, mask, p, precision=prec)
    known = mask == 0
    np.testing.assert_array_equal(out[known], img[known].astype(np.float64))
    assert (om[mask == 1] == 2).all() and (om[known] == 0).all()
    assert np.isfinite(out).all()
    assert rep.unconcealed_blocks == []
    assert rep.blocks_processed == int((P.lost_per_block(P.build_grid(1920, 1080, 4), mask) > 0).sum())
    # fp32 agrees with the fp64 path on the same frame (statistically, see FP32_PSNR_DB)
    out64, _, _ = P.conceal(img, mask, p, precision="fp64")
    lost = mask == 1
    truth = img.astype(np.float64)
    assert abs(psnr(truth, out, mask) - psnr(truth, out64, mask)) <= FP32_PSNR_DB
    assert np.mean(np.abs(out[lost] - out64[lost]) <= 0.5) >= 0.6


@pytest.mark.parametrize("cfg,B,F,order", [(2, 4, 64, "optimized"), (2, 4, 64, "linescan"),
                                           (5, 2, 32, "optimized")])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_dataflow_equals_level_launches(cfg, B, F, order, prec):
    """The persistent dataflow launch and the per-level launches compute the
    same function (every block reads only lower-rank, completed blocks)."""
    from paper_2207_00233_b200 import _lib

    img, mask = synth.config_scene(cfg)
    if cfg == 5:
        img, mask = img[:256, :384].copy(), mask[:256, :384].copy()
    p = P.FseParams(d=14, iterations=40, block_size=B, fft_size=F)
    L = _lib.lib()
    try:
        L.fse_set_dataflow(1)
        a, am, _ = P.conceal(img, mask, p, order, precision=prec)
        L.fse_set_dataflow(0)
        b, bm, _ = P.conceal(img, mask, p, order, precision=prec)
    finally:
        L.fse_set_dataflow(0)
    assert a.tobytes() == b.tobytes()
    np.testing.assert_array_equal(am, bm)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_frame_groups_equal_one_launch_sequence(prec):
    """Frame groups on forked streams (fse_set_groups) compute the same images
    and masks as one level-launch sequence over all frames."""
    from paper_2207_00233_b200 import _lib

    sc = [synth.config_scene(4, f) for f in range(3)]
    imgs = np.stack([s[0][:160, :224] for s in sc])
    msks = np.stack([s[1][:160, :224] for s in sc])
    p = P.FseParams(d=14, iterations=30, block_size=4, fft_size=64)
    L = _lib.lib()
    outs = []
    try:
        for g in (1, 2, 3):
            assert L.fse_set_groups(g) == 0
            o, m, _ = P.conceal_batch(imgs, msks, p, precision=prec, reports=False)
            outs.append((o.tobytes(), m.tobytes()))
    finally:
        L.fse_set_groups(2)
    assert outs[0] == outs[1] == outs[2]
    assert L.fse_set_groups(0) != 0 and L.fse_set_groups(9) != 0


@pytest.mark.parametrize("B,F", [(2, 32), (4, 64), (8, 128)])
def test_config5_block_sizes_fp32_fast_path(B, F):
    """fp32 fast kernels at F = 32 / 64 / 128 against the fp64 path on a crop of
    BASELINE config 5 (statistical parity, FP32_PSNR_DB)."""
    img, mask = synth.config_scene(5)
    img, mask = img[:128, :192].copy(), mask[:128, :192].copy()
    p = P.FseParams(d=14, iterations=60, block_size=B, fft_size=F)
    o32, m32, _ = P.conceal(img, mask, p, precision="fp32")
    o64, m64, _ = P.conceal(img, mask, p, precision="fp64")
    np.testing.assert_array_equal(m32, m64)
    truth = img.astype(np.float64)
    assert abs(psnr(truth, o32, mask) - psnr(truth, o64, mask)) <= FP32_PSNR_DB
    assert np.isfinite(o32).all()


@pytest.mark.parametrize("prec,world", [("fp64", 2), ("fp32", 3)])
def test_strip_shards_on_one_gpu_equal_whole_frame(prec, world):
    """The C-ABI shard sessions (fse_shard_*) of a row-band partition, stepped
    level by level with the halo copies of paper_2207_00233_b200.strips (done
    here as device copies between the bands' images), reproduce the
    whole-frame result bit for bit.  The NCCL transport itself is covered on
    CPU by tests/test_strips.py."""
    import torch

    from paper_2207_00233_b200 import strips

    img, mask = synth.config_scene(5)
    img, mask = img[:256, :384].copy(), mask[:256, :384].copy()
    H = img.shape[0]
    p = P.FseParams(d=14, iterations=30, block_size=4, fft_size=64)
    want, want_m, _ = P.conceal(img, mask, p, precision=prec)
    plan = P.build_plan(mask, p)
    R = strips.halo_rows(p)
    processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(plan.rows, plan.cols)
    bands = strips.band_partition(processed.sum(axis=1), world, R)
    tdt = torch.float32 if prec == "fp32" else torch.float64
    imgs = [torch.from_numpy(img).cuda().to(tdt) for _ in range(world)]
    msk = torch.from_numpy(mask).cuda()
    outs = [torch.zeros_like(msk) for _ in range(world)]
    exs = [strips.ShardExecutor(plan, bands[r], imgs[r], msk, outs[r], p, prec) for r in range(world)]
    levels = plan.levels()
    for r in range(world):
        np.testing.assert_array_equal(exs[r].flags, strips.edge_flags(levels, plan.cols, bands[r], R))
    flags_all = [e.flags for e in exs]
    for l in range(plan.n_levels):
        for e in exs:
            e.run(l)
        for r in range(world):
            sends, _ = strips.exchange_plan(r, world, bands, flags_all, l, R, p.block_size, H)
            for peer, y0, y1 in sends:
                imgs[peer][y0:y1].copy_(imgs[r][y0:y1])
    for e in exs:
        e.close()
    got = np.zeros_like(want)
    got_m = np.zeros_like(want_m)
    for r, (lo, hi) in enumerate(bands):
        y0, y1 = lo * p.block_size, min(H, hi * p.block_size)
        got[y0:y1] = imgs[r][y0:y1].double().cpu().numpy()
        got_m[y0:y1] = outs[r][y0:y1].cpu().numpy()
    assert got.tobytes() == want.tobytes()
    np.testing.assert_array_equal(got_m, want_m)


def test_conceal_strips_single_rank_equals_conceal():
    from paper_2207_00233_b200 import strips

    img, mask = synth.config_scene(5)
    img, mask = img[:128, :256].copy(), mask[:128, :256].copy()
    p = P.FseParams(d=14, iterations=30, block_size=4, fft_size=64)
    want, want_m, _ = P.conceal(img, mask, p, precision="fp64")
    got, got_m = strips.conceal_strips(img, mask, p, precision="fp64")
    assert got.tobytes() == want.tobytes()
    np.testing.assert_array_equal(got_m, want_m)


@pytest.mark.parametrize("config,B,F,iters", [(3, 4, 64, 200), (5, 4, 64, 100), (5, 2, 32, 100),
                                              (5, 8, 128, 100), (4, 4, 64, 100)])
def test_full_size_fp64_blocks_match_oracle_on_their_snapshots(config, B, F, iters):
    """Full-size parity without a full-size CPU run: every block's window is a
    pure function of the original mask, the plan ranks and the final values of
    lower-rank blocks (written once, never changed).  So for a seeded sample of
    blocks, re-fitting the snapshot rebuilt from the GPU's own output with the
    oracle must reproduce the GPU's picks and samples (fp64: identical canonical
    picks, samples within 1e-6)."""
    from helpers import block_owner

    img, mask = synth.config_scene(config)
    H, W = mask.shape
    p = P.FseParams(d=14, iterations=iters, block_size=B, fft_size=F)
    out, _, rep, picks = P.conceal(img, mask, p, precision="fp64", return_picks=True)
    plan = P.build_plan(mask, p)
    ranks = plan.ranks()
    owner = block_owner(H, W, B)
    op = O.Params(d=14, rho=0.8, delta=0.2, gamma=0.5, iterations=iters, block_size=B, fft_size=(F, F))
    processed = np.flatnonzero(ranks != np.iinfo(np.int32).max)
    rng = np.random.default_rng(config * 10 + B)
    sample = rng.choice(processed, size=min(24, processed.size), replace=False)
    cols = plan.cols
    for b in sample.tolist():
        r, c = divmod(b, cols)
        r0, r1, c0, c1 = r * B, min(r * B + B, H), c * B, min(c * B + B, W)
        wr0, wr1, wc0, wc1 = max(0, r0 - 14), min(H, r1 + 14), max(0, c0 - 14), min(W, c1 + 14)
        sub = mask[wr0:wr1, wc0:wc1]
        own = owner[wr0:wr1, wc0:wc1]
        lost = sub == O.LOST
        cls = np.where(sub == O.RECONSTRUCTED, O.AREA_R, O.AREA_A).astype(np.uint8)
        earlier = ranks[own] < ranks[b]
        cls[lost & (own != b) & earlier] = O.AREA_R
        cls[lost & (own != b) & ~earlier] = O.AREA_BO
        cls[lost & (own == b)] = O.AREA_BI
        vals = np.where(lost & ~((own != b) & earlier), 0.0, out[wr0:wr1, wc0:wc1])
        vals = np.where(~lost, img[wr0:wr1, wc0:wc1].astype(np.float64), vals)
        blk, opk = O.extrapolate(vals, cls, (r0 - wr0, r1 - wr0, c0 - wc0, c1 - wc0), op, "c",
                                 want_picks=True)
        assert O.canonical_picks(picks[b], (F, F)) == O.canonical_picks(opk, (F, F)), b
        lb = mask[r0:r1, c0:c1] == O.LOST
        assert np.max(np.abs(out[r0:r1, c0:c1][lb] - blk[lb])) <= 1e-6, b


def test_quantize_psnr_epilogue_matches_reference_semantics():
    """fse_quantize_psnr: save_pgm rounding (image.py:79-88) and evalkit.psnr
    (evalkit.py:67-81) over non-KNOWN samples, on device, for fp32 and fp64."""
    import torch

    rng = np.random.default_rng(3)
    n, H, W = 3, 40, 56
    truth = rng.integers(0, 256, (n, H, W)).astype(np.uint8)
    mask = (rng.uniform(size=(n, H, W)) < 0.3).astype(np.uint8)
    mask[1][mask[1] == 1] = 2  # post-concealment mask states count too
    vals = truth + rng.normal(0, 9, (n, H, W))
    vals[0, 0, :6] = [-3.0, 0.5, 1.5, 254.5, 255.49, 300.0]  # clamping and half-up ties
    for dt in (torch.float32, torch.float64):
        x = torch.from_numpy(vals).to(dt)
        u8, ps = P.quantize_psnr_device(x.cuda(), torch.from_numpy(truth).cuda(), torch.from_numpy(mask).cuda())
        xv = x.double().numpy()
        np.testing.assert_array_equal(u8.cpu().numpy(), np.floor(np.clip(xv, 0, 255) + 0.5).astype(np.uint8))
        for f in range(n):
            want = psnr(truth[f].astype(np.float64), xv[f], mask[f])
            assert abs(ps[f] - want) <= 1e-9 * abs(want)


@pytest.mark.parametrize("shape,B,F,prec", [((37, 53), 4, 64, "fp64"), ((10, 12), 4, 32, "fp64"),
                                            ((37, 53), 4, 64, "fp32"), ((70, 45), 8, 128, "fp32"),
                                            ((70, 45), 8, 128, "fp64"), ((33, 31), 2, 32, "fp64")])
def test_ragged_and_tiny_frames_fast_path_vs_oracle(shape, B, F, prec):
    """Ragged block grids and frames smaller than a window through the fast
    kernels, against the oracle pipeline (fp64: 1e-6; fp32: PSNR parity)."""
    H, W = shape
    rng = np.random.default_rng(H * W + B)
    yy, xx = np.mgrid[0:H, 0:W]
    img = np.clip(128 + 50 * np.sin(0.21 * xx + 0.13 * yy) + rng.normal(0, 2, shape), 0, 255).round()
    mask = np.zeros(shape, np.uint8)
    mask[rng.uniform(size=shape) < 0.0] = 1
    for _ in range(4):
        r0, c0 = int(rng.integers(0, H - 3)), int(rng.integers(0, W - 3))
        mask[r0:r0 + int(rng.integers(2, 9)), c0:c0 + int(rng.integers(2, 9))] = 1
    img[mask == 1] = 0
    p = P.FseParams(d=14, iterations=25, block_size=B, fft_size=F)
    out, om, rep = P.conceal(img, mask, p, precision=prec)
    o_img, o_msk, o_rep = O.conceal(img, mask, O.Params(d=14, iterations=25, block_size=B, fft_size=(F, F)),
                                    "optimized", kernel="auto")
    assert rep.batches == o_rep.batches
    np.testing.assert_array_equal(om, o_msk)
    if prec == "fp64":
        assert np.max(np.abs(out - o_img)) <= 1e-6
    else:
        truth = img.astype(np.float64)
        assert abs(psnr(truth, out, mask) - psnr(truth, o_img, mask)) <= FP32_PSNR_DB


def test_fp32_guard_redo_everything_matches_fp64():
    """fse_set_guard(1, 0) hands every fp32 window to the fp64 redo kernel
    (fse_fast_redo_kernel): the result is the fp64 path's up to fp32 storage of
    the image (the guard machinery)."""
    from paper_2207_00233_b200 import _lib

    img, mask = synth.config_scene(2)
    img, mask = img[:192, :256].copy(), mask[:192, :256].copy()
    p = P.FseParams(d=14, iterations=60, block_size=4, fft_size=64)
    L = _lib.lib()
    try:
        L.fse_set_guard(1.0, 0.0)
        L.fse_guard_redo_count(1)
        L.fse_timing_enable(1)
        g32, m32, rep = P.conceal(img, mask, p, precision="fp32")
        L.fse_timing_enable(0)
        L.fse_timing_read(None, None, None)
        redone = int(L.fse_guard_redo_count(1))
    finally:
        L.fse_set_guard(-1.0, 0.0)
        L.fse_timing_enable(0)
    o64, m64, _ = P.conceal(img, mask, p, precision="fp64")
    assert redone == rep.blocks_processed
    np.testing.assert_array_equal(m32, m64)
    assert np.max(np.abs(g32 - o64)) <= 1e-3


@pytest.mark.parametrize("cfg,B,F", [(3, 4, 64), (5, 2, 32)])
def test_tracked_and_lazy_argmax_identical(cfg, B, F):
    """fp32 level launches pick the argmax form by width (fse_set_track_below):
    the tracked form (best bin carried per thread, one barrier) and the lazy
    form (running maximum, second barrier) find the same first maximum, so the
    frames are bit-identical."""
    from paper_2207_00233_b200 import _lib

    img, mask = synth.config_scene(cfg)
    img, mask = img[:192, :320].copy(), mask[:192, :320].copy()
    p = P.FseParams(d=14, iterations=60, block_size=B, fft_size=F)
    L = _lib.lib()
    outs = []
    try:
        for below in (1 << 30, 0):  # always tracked, always lazy
            assert L.fse_set_track_below(below) == 0
            o, m, _ = P.conceal(img, mask, p, precision="fp32")
            outs.append((o.tobytes(), m.tobytes()))
    finally:
        L.fse_set_track_below(148 * 16)
    assert outs[0] == outs[1]
    assert L.fse_set_track_below(-1) != 0


@pytest.mark.parametrize("world,B", [(2, 4), (3, 2)])
def test_strips_fused_peer_exchange_multi_process(world, B):
    """Strip sharding over `world` processes (one GPU here; CUDA IPC maps the
    neighbours' frames and flags): the fused halo exchange (peer stores in the
    level kernel, device-flag ordering, one shard call per frame) and the
    per-level collective exchange both reproduce the whole-frame conceal bit
    for bit, twice in a row (flag epochs)."""
    import subprocess
    import sys

    drv = os.path.join(os.path.dirname(os.path.abspath(__file__)), "strips_p2p_driver.py")
    r = subprocess.run([sys.executable, drv, str(world), "5", str(B)], capture_output=True, text=True,
                       timeout=400)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("prec,batch,depth", [("fp32", 3, 2), ("fp64", 4, 3)])
def test_conceal_stream_equals_per_frame(prec, batch, depth):
    """ConcealStream (frames pushed one at a time, batched, upload / plan /
    levels / download of neighbouring batches overlapped) returns, in push
    order, exactly what conceal() gives per frame -- including a partial last
    batch and more batches than slots (backpressure)."""
    nf = 9
    frames = [synth.synthetic_frame(96, 160, 70 + f, 6, 3) for f in range(nf)]
    masks = [synth.loss_mask(96, 160, "mixed", 0.25, 80 + f) for f in range(nf)]
    p = P.FseParams(d=14, iterations=30, block_size=4, fft_size=64)
    got = []
    with P.ConcealStream(p, (96, 160), batch=batch, precision=prec, depth=depth,
                         in_dtype=np.float64 if prec == "fp64" else np.uint8) as st:
        for f in range(nf):
            got += st.push(frames[f], masks[f])
        got += st.flush()
    assert len(got) == nf
    for f in range(nf):
        one, om, _ = P.conceal(frames[f], masks[f], p, precision=prec)
        assert got[f][0].astype(np.float64).tobytes() == one.tobytes()
        np.testing.assert_array_equal(got[f][1], om)


# ---- full-size reference goldens (tests/golden/make_golden_large.py) ----------

LARGE = ["cfg3", "cfg4f0", "cfg5crop", "cfg3def"]


@pytest.mark.parametrize("name", LARGE)
def test_large_golden_fp64_identical_picks(golden, name):
    """BASELINE config 3, config 4 frame 0, a 768x1024 crop of the 4K config-5
    frame, and config 3 with the reference's DEFAULT parameters (the drop-in
    call, DFT = window size): fp64 canonical pick sequence of EVERY block
    identical to the reference's (64-bit hash of each sequence, full sequences
    of every 16th block), every lost sample within 1e-6, batches and mask equal."""
    from helpers import canonical_fold, large_case, pick_hash, window_shapes

    g = golden(f"large_{name}.npz")
    img, mask, kw, fft = large_case(g)
    p = P.FseParams(fft_size=fft, **kw)
    out, msk, rep, picks = P.conceal(img, mask, p, "optimized", precision="fp64", return_picks=True)
    assert rep.batches == csr(g["batch_ptr"], g["batch_blocks"])
    assert rep.unconcealed_blocks == g["unconcealed"].tolist()
    assert int(msk.astype(np.int64).sum()) == int(g["out_mask_sum"])
    lost = mask == 1
    err = np.abs(out[lost] - g["lost_values"])
    assert float(err.max()) <= 1e-6, (float(err.max()), int((err > 1e-6).sum()))
    blocks = g["pick_blocks"]
    H, W = mask.shape
    if fft is None:
        F1, F2 = window_shapes(H, W, kw["block_size"], kw["d"], blocks)
    else:
        F1, F2 = fft
    canon = canonical_fold(picks[blocks], F1, F2)
    bad = np.flatnonzero(pick_hash(canon) != g["pick_hash"])
    assert bad.size == 0, f"{bad.size} blocks differ, first {blocks[bad[:5]].tolist()}"
    idx = np.searchsorted(blocks, g["sample_blocks"])
    np.testing.assert_array_equal(canon[idx], g["sample_picks"].astype(np.int64))


def test_conceal_batch_64_frames_fp64_matches_reference_frame0(golden):
    """The bench path (conceal_batch over BASELINE config 4's 64 frames, every
    frame's level in one merged launch, staged chunks) in fp64: frame 0 equals
    the reference's frame 0 within 1e-6; every frame equals per-frame conceal()
    for a sample of frames."""
    from concurrent.futures import ThreadPoolExecutor

    from helpers import large_case

    g = golden("large_cfg4f0.npz")
    img0, mask0, kw, fft = large_case(g)
    with ThreadPoolExecutor(8) as ex:
        scenes = list(ex.map(lambda f: synth.config_scene(4, f), range(64)))
    imgs = np.stack([s[0] for s in scenes])
    msks = np.stack([s[1] for s in scenes])
    assert np.array_equal(imgs[0], img0) and np.array_equal(msks[0], mask0)
    p = P.FseParams(fft_size=fft, **kw)
    out, om, _ = P.conceal_batch(imgs, msks, p, "optimized", "fp64", reports=False)
    lost = mask0 == 1
    assert float(np.max(np.abs(out[0][lost] - g["lost_values"]))) <= 1e-6
    assert int(om[0].astype(np.int64).sum()) == int(g["out_mask_sum"])
    for f in (1, 31, 63):
        o1, m1, _ = P.conceal(imgs[f], msks[f], p, "optimized", precision="fp64")
        np.testing.assert_array_equal(out[f], o1)
        np.testing.assert_array_equal(om[f], m1)


@pytest.mark.gpu
def test_device_entry_points_reject_mismatched_buffers():
    """run_frames_device / ShardExecutor hand raw pointers to the C ABI: a
    working image of the wrong type (fp32 buffer for the fp64 path), shape or
    layout is rejected before any launch, never read as the wrong type."""
    import torch
    from paper_2207_00233_b200 import strips

    img, mask = synth.config_scene(1)
    p = P.FseParams(d=14, iterations=5, block_size=4, fft_size=64)
    plan = P.build_plan(mask, p)
    m = torch.from_numpy(mask).cuda()
    out = torch.empty_like(m)
    f32 = torch.from_numpy(img).cuda().float()
    with pytest.raises(ValueError, match="precision"):
        P.run_frames_device([plan], [f32], [m], [out], p, "fp64")
    with pytest.raises(ValueError, match="precision"):
        strips.ShardExecutor(plan, (0, plan.rows), f32, m, out, p, "fp64")
    f64 = f32.double()
    with pytest.raises(ValueError, match="does not match"):
        P.run_frames_device([plan], [f64[:-8]], [m[:-8]], [out], p, "fp64")
    with pytest.raises(ValueError, match="contiguous"):
        P.run_frames_device([plan], [f64.t()], [m.t()], [out], p, "fp64")
    P.run_frames_device([plan], [f64], [m], [out], p, "fp64")  # the matching call runs
    torch.cuda.synchronize()


@pytest.mark.parametrize("prec,B,F", [("fp64", 4, 64), ("fp32", 4, 64), ("fp64", 8, 128), ("fp64", 16, None)])
def test_level_balancing_never_changes_a_bit(prec, B, F, monkeypatch):
    """fse_plan_rebalance only changes in which launch a block runs: with it on
    (the default of one-frame calls) and off, conceal() returns identical bytes,
    batches (conceal.py:148-163) and picks -- on a frame whose plan really has
    wide first levels and a narrow tail, so that blocks do move."""
    from paper_2207_00233_b200 import synth

    img, mask = synth.config_scene(3)
    img, mask = img[:540, :960].astype(np.float64), mask[:540, :960].copy()
    img[mask == 1] = 0
    p = P.FseParams(d=14 if F else 16, iterations=12, block_size=B, fft_size=F)
    plan = P.build_plan(mask, p)
    widths = [len(l) for l in plan.levels()]
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    moved = plan.rebalance(sms, 0)
    if F == 64:
        assert max(widths) > sms and min(widths) < sms and moved > 0
    monkeypatch.setenv("FSE_BALANCE", "0")
    off = P.conceal(img, mask, p, precision=prec, return_picks=True)
    monkeypatch.setenv("FSE_BALANCE", "1")
    on = P.conceal(img, mask, p, precision=prec, return_picks=True)
    assert on[0].tobytes() == off[0].tobytes() and on[1].tobytes() == off[1].tobytes()
    assert on[2].batches == off[2].batches and on[2].blocks_processed == off[2].blocks_processed
    assert on[3].tobytes() == off[3].tobytes()
