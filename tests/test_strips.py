"""Spatial strip sharding (BASELINE config 5) on CPU: the band
partition, the halo exchange schedule, and the full level/halo protocol of
paper_2207_00233_b200.strips run by two gloo ranks with the oracle standing in
for the device kernel — bit-identical to one process doing the whole frame."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2207_00233_b200 as P
from helpers import block_owner, emulate_block, emulate_levels
from oracle import oracle as O
from paper_2207_00233_b200 import strips, synth

H, W, B, D, ITERS, FFT = 96, 128, 4, 14, 12, 64


def _scene():
    img = synth.synthetic_frame(H, W, 77, 6, 3).astype(np.float64)
    mask = synth.loss_mask(H, W, "burst2d", 0.3, 78)
    img[mask == 1] = 0.0
    return img, mask


def _params():
    return P.FseParams(d=D, iterations=ITERS, block_size=B, fft_size=FFT)


def test_band_partition_covers_rows_and_balances():
    rng = np.random.default_rng(0)
    for rows, world, R in [(24, 2, 4), (540, 8, 4), (135, 4, 2), (1080, 8, 7), (9, 3, 3)]:
        w = rng.integers(0, 60, rows)
        bands = strips.band_partition(w, world, R)
        assert bands[0][0] == 0 and bands[-1][1] == rows
        assert all(b[0] < b[1] for b in bands)
        assert all(bands[k][1] == bands[k + 1][0] for k in range(world - 1))
        assert all(b[1] - b[0] >= max(R, 1) for b in bands)
        loads = [w[a:b].sum() for a, b in bands]
        assert max(loads) - min(loads) <= 2 * w.max() + 1
    with pytest.raises(ValueError):
        strips.band_partition(np.ones(5), 3, 2)


def test_exchange_schedule_is_symmetric():
    img, mask = _scene()
    plan = P.build_plan(mask, _params())
    levels = plan.levels()
    R = strips.halo_rows(_params())
    for world in (2, 3):
        processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(plan.rows, plan.cols)
        bands = strips.band_partition(processed.sum(axis=1), world, R)
        flags = [strips.edge_flags(levels, plan.cols, b, R) for b in bands]
        for l in range(len(levels)):
            plans = [strips.exchange_plan(r, world, bands, flags, l, R, B, H) for r in range(world)]
            for r in range(world):
                for peer, y0, y1 in plans[r][0]:  # every send has the matching recv
                    assert (r, y0, y1) in plans[peer][1]
                for peer, y0, y1 in plans[r][1]:
                    assert (r, y0, y1) in plans[peer][0]


class EmuExecutor:
    """The device kernel's semantics on the CPU (oracle kernel, rank-based
    classes), restricted to one band."""

    def __init__(self, plan, band, image, mask, params):
        self.levels = plan.levels()
        self.ranks = plan.ranks()
        self.cols = plan.cols
        self.band = band
        self.image = image
        self.mask = mask
        self.owner = block_owner(H, W, B)
        self.p = O.Params(d=params.d, rho=params.rho, delta=params.delta, gamma=params.gamma,
                          iterations=params.iterations, block_size=B, fft_size=(FFT, FFT))
        self.n_levels = len(self.levels)
        self.flags = strips.edge_flags(self.levels, self.cols, band, strips.halo_rows(params))

    def run(self, level, level_hi=None):
        lo, hi = self.band
        for lv in range(level, level + 1 if level_hi is None else level_hi):
            for b in self.levels[lv]:
                if lo <= b // self.cols < hi:
                    emulate_block(self.image, self.mask, b, self.ranks, self.owner, B, self.p)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img, mask = _scene()
    params = _params()
    # rank 0 plans, the others import the broadcast bytes (the GPU default)
    plan = strips.broadcast_plan(mask, params, "optimized", rank, dist, None, 0)
    local = P.build_plan(mask, params)
    assert plan.batches() == local.batches() and plan.levels() == local.levels()
    assert (plan.ranks() == local.ranks()).all() and plan.unconcealed() == local.unconcealed()
    R = strips.halo_rows(params)
    processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(plan.rows, plan.cols)
    bands = strips.band_partition(processed.sum(axis=1), world, R)
    image = torch.from_numpy(img.copy())
    ex = EmuExecutor(plan, bands[rank], image, mask, params)
    t = torch.from_numpy(ex.flags.astype(np.int64))
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    flags_all = [g.numpy() for g in gathered]
    sent = strips.run_levels(ex, image, rank, world, bands, flags_all, ex.n_levels, R, B, H, dist)
    lo, hi = bands[rank]
    if rank == 0:
        for r in range(1, world):
            a, b = bands[r][0] * B, min(H, bands[r][1] * B)
            dist.recv(image[a:b], r)
        out.put((image.numpy().copy(), sent))
    else:
        dist.send(image[lo * B:min(H, hi * B)].contiguous(), 0)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_strip_protocol_equals_whole_frame(world):
    img, mask = _scene()
    params = _params()
    plan = P.build_plan(mask, params)
    want, _ = emulate_levels(img, mask, B, D, params.rho, params.delta, params.gamma, ITERS, (FFT, FFT),
                             plan.ranks(), plan.levels())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.spawn(_worker, args=(world, _free_port(), q), nprocs=world, join=False)
    got, sent = q.get(timeout=300)  # read before join: a large item blocks the child's exit
    while not pc.join():
        pass
    assert sent > 0  # halos actually crossed ranks
    np.testing.assert_array_equal(got, want)
