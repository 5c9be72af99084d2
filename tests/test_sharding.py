"""Frame-parallel sharding (BASELINE config 4) on CPU: two gloo
ranks split the frames, build their C++ plans, and the all-reduced work
equals the single-process total.  No GPU: plans are host C++ only."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth

FRAMES = 6
H, W = 96, 160


def _scene(f):
    img = synth.synthetic_frame(H, W, 4000 + f, 6, 3)
    mask = synth.loss_mask(H, W, "mixed", 0.2, 5000 + f)
    return img, mask


def _params():
    return P.FseParams(d=14, iterations=10, block_size=4, fft_size=64)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    ids = bench.frame_ids(4, FRAMES, rank, world)
    masks = [_scene(f)[1] for f in ids]
    plans = P.build_plans(masks, _params(), "optimized", 2)
    t = torch.tensor([sum(p.n_processed for p in plans), len(ids)], dtype=torch.float64)
    dist.all_reduce(t)
    got = [None] * world
    dist.all_gather_object(got, ids)
    if rank == 0:
        out.put((t.tolist(), got))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_frame_ids_partition():
    for world in (1, 2, 3, 4, 8):
        seen = [f for r in range(world) for f in bench.frame_ids(4, 64, r, world)]
        assert seen == list(range(64))
        sizes = [len(bench.frame_ids(4, 64, r, world)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
def test_two_gloo_ranks_cover_the_batch_once():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q), nprocs=2, join=True)
    (blocks, nframes), ids = q.get(timeout=60)
    assert sorted(f for r in ids for f in r) == list(range(FRAMES))
    assert not set(ids[0]) & set(ids[1])
    plans = P.build_plans([_scene(f)[1] for f in range(FRAMES)], _params(), "optimized", 2)
    assert blocks == sum(p.n_processed for p in plans)
    assert nframes == FRAMES


def test_conceal_batch_chunk_bounds(monkeypatch):
    """conceal_batch's staged pipeline covers every frame exactly once, in order."""
    from paper_2207_00233_b200.conceal import _chunk_bounds

    for n in (1, 2, 3, 4, 5, 9, 12, 15, 16, 63, 64, 100):
        b = _chunk_bounds(n)
        assert b[0] == 0 and b[-1] == n
        assert all(x < y for x, y in zip(b, b[1:]))
        assert len(b) == (2 if n < 12 else 3 if n < 16 else 4)
    monkeypatch.setenv("FSE_CHUNKS", "0.0625,0.125,0.6875,0.125")
    for n in (1, 5, 64):
        b = _chunk_bounds(n)
        assert b[0] == 0 and b[-1] == n and all(x < y for x, y in zip(b, b[1:]))
    assert _chunk_bounds(64) == [0, 4, 12, 56, 64]
