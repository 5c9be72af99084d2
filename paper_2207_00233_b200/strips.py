"""Spatial strip sharding of one large frame across GPUs (BASELINE config 5).

One process per GPU; every rank builds the same global plan (the C++ planner
is deterministic), so ranks, batches and dependency levels agree everywhere.
Rank r owns a band of block rows [lo_r, hi_r), balanced by lossy-block count.
Level by level, each rank fits the blocks of its band and then swaps halos with
its neighbours: the window of a block reaches R = ceil(d/B) block rows, so the
image rows of the R block rows at a band edge are sent to the neighbouring rank
whenever that level wrote blocks there.  Masks and ranks never change (the
snapshot semantics is rank-based), so only image samples move.
The reference has no counterpart: its only parallelism is a thread pool over
one batch (fsefill/conceal.py:146-153).

The level loop and the exchange schedule are written against a small executor
interface so the same protocol runs on GPUs (ShardExecutor, C ABI fse_shard_*,
NCCL point-to-point) and, in tests, on CPU ranks over gloo with an emulated
kernel.  The default GPU transport fuses the exchange into the kernel instead
(PeerLink): band-edge blocks are stored straight into the neighbour's frame
over NVLink and levels are ordered by device flags, so a shard's whole level
sequence is one call.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .conceal import DeviceContext, Plan, balance_for_device, build_plan
from .fse import FseParams


_HOST_GROUPS: dict = {}


def host_group(dist, group=None):
    """A gloo group over the same ranks (host-side collectives: plan bytes,
    flags), created once; `group` itself when it is already gloo."""
    if dist.get_backend(group) == "gloo":
        return group
    key = None if group is None else tuple(dist.get_process_group_ranks(group))
    g = _HOST_GROUPS.get(key)
    if g is None:
        g = dist.new_group(ranks=None if key is None else list(key), backend="gloo")
        _HOST_GROUPS[key] = g
    return g


def broadcast_plan(mask, params: FseParams, order: str, rank: int, dist, group=None, src: int = 0,
                   plan_threads: int = 0, precision: str | None = None):
    """Plan the frame on rank `src` only and broadcast the plan's bytes
    (fse_plan_export / fse_plan_import) -- instead of every rank planning the
    same frame with its share of the host CPUs.  `group` must carry CPU
    tensors (gloo), so waiting ranks block in the transport, not on a GPU
    stream.  `plan_threads` is the planning rank's thread count (0 = 3/4 of
    the usable CPUs: the other ranks are idle meanwhile).  With `precision` the
    plan's levels are balanced for the planning rank's device before the
    broadcast (conceal.balance_for_device)."""
    import os

    import torch

    if rank == src:
        T = plan_threads or max(1, (3 * len(os.sched_getaffinity(0))) // 4)
        plan = build_plan(mask, params, order, plan_threads=T)
        if precision is not None:
            balance_for_device(plan, params, precision, world=dist.get_world_size(group))
        data = plan.to_bytes()
        n = torch.tensor([len(data)], dtype=torch.int64)
    else:
        n = torch.zeros(1, dtype=torch.int64)
    dist.broadcast(n, src, group=group)
    if rank == src:
        t = torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy())
    else:
        t = torch.empty(int(n.item()), dtype=torch.uint8)
    dist.broadcast(t, src, group=group)
    return plan if rank == src else Plan.from_bytes(t.numpy().tobytes())


def halo_rows(params: FseParams) -> int:
    """Dependency radius in block rows: a window spans block +- d samples."""
    return -(-params.d // params.block_size) if params.d > 0 else 0


def band_partition(lossy_per_row, world: int, R: int) -> list:
    """Split block rows into `world` contiguous bands with about equal lossy-block
    counts; every band keeps at least max(R, 1) rows so halos come only from the
    adjacent ranks."""
    rows = len(lossy_per_row)
    min_rows = max(R, 1)
    if world < 1:
        raise ValueError("world must be >= 1")
    if world * min_rows > rows:
        raise ValueError(f"{rows} block rows cannot be split into {world} bands of >= {min_rows} rows")
    w = np.asarray(lossy_per_row, dtype=np.float64) + 1e-3  # empty rows still cost a little
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        c = int(np.searchsorted(cum, target))
        lo_ok = cuts[-1] + min_rows
        hi_ok = rows - (world - k) * min_rows
        cuts.append(min(max(c, lo_ok), hi_ok))
    cuts.append(rows)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def edge_flags(level_blocks, cols: int, band, R: int) -> np.ndarray:
    """Per level: bit 0 if the band wrote blocks within R rows of its top edge,
    bit 1 for the bottom edge (what fse_shard_levels reports)."""
    lo, hi = band
    out = np.zeros(len(level_blocks), dtype=np.int32)
    for l, blocks in enumerate(level_blocks):
        r = np.asarray(blocks, dtype=np.int64) // cols
        r = r[(r >= lo) & (r < hi)]
        if r.size:
            out[l] = int((r < lo + R).any()) | (int((r >= hi - R).any()) << 1)
    return out


def exchange_plan(rank: int, world: int, bands, flags_all, level: int, R: int, B: int, H: int):
    """(sends, recvs) of one level: lists of (peer, y0, y1) image-row ranges."""
    lo, hi = bands[rank]
    sends, recvs = [], []
    if rank > 0:
        if flags_all[rank][level] & 1:
            sends.append((rank - 1, lo * B, min(H, (lo + R) * B)))
        if flags_all[rank - 1][level] & 2:
            recvs.append((rank - 1, max(0, (lo - R) * B), lo * B))
    if rank < world - 1:
        if flags_all[rank][level] & 2:
            sends.append((rank + 1, max(0, (hi - R) * B), min(H, hi * B)))
        if flags_all[rank + 1][level] & 1:
            recvs.append((rank + 1, hi * B, min(H, (hi + R) * B)))
    return sends, recvs


def run_levels(executor, image, rank: int, world: int, bands, flags_all, n_levels: int, R: int,
               B: int, H: int, dist, group=None) -> int:
    """The protocol: run each level of the own band, then swap the halos the
    level changed.  `image` is the rank's full-frame tensor (device or host);
    row slices are contiguous views, sent and received in place.  Returns the
    number of halo messages this rank sent."""
    sent = 0
    if world == 1:  # nothing to exchange: every level in one C++ call
        if n_levels:
            executor.run(0, n_levels)
        return 0
    for l in range(n_levels):
        executor.run(l)
        sends, recvs = exchange_plan(rank, world, bands, flags_all, l, R, B, H)
        if not sends and not recvs:
            continue
        if getattr(image, "is_cuda", False) and dist.get_backend(group) == "gloo":
            # gloo moves host memory only: stage the halo rows through the host
            # (functional runs of several ranks on one GPU; NCCL sends in place)
            rbufs = [(image[y0:y1], image[y0:y1].cpu()) for _, y0, y1 in recvs]
            ops = [dist.P2POp(dist.isend, image[y0:y1].cpu(), peer, group) for peer, y0, y1 in sends]
            ops += [dist.P2POp(dist.irecv, hb, peer, group) for (peer, _, _), (_, hb) in zip(recvs, rbufs)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for dv, hb in rbufs:
                dv.copy_(hb)
        else:
            ops = [dist.P2POp(dist.isend, image[y0:y1], peer, group) for peer, y0, y1 in sends]
            ops += [dist.P2POp(dist.irecv, image[y0:y1], peer, group) for peer, y0, y1 in recvs]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        sent += len(sends)
    return sent


class ShardExecutor:
    """GPU executor: one fse_shard_* session over a band of the rank's frame."""

    def __init__(self, plan, band, image_dev, mask_dev, mask_out_dev, params: FseParams,
                 precision: str, stream=None):
        import torch

        from .conceal import check_device_frames

        check_device_frames([image_dev], [mask_dev], [plan], precision, params.block_size)
        self.stream = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        dim = max(plan.max_wr, plan.max_wc, 1)
        self._decay = DeviceContext.decay(params, dim)
        code = _lib.FSE_F64 if precision == "fp64" else _lib.FSE_F32
        pc = params.to_c()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().fse_shard_open(
            plan.handle, band[0], band[1], image_dev.data_ptr(), mask_dev.data_ptr(),
            mask_out_dev.data_ptr() if mask_out_dev is not None else None, ctypes.byref(pc), code,
            self._decay.data_ptr(), dim, self.stream, ctypes.byref(h)))
        self.handle = h
        n = ctypes.c_int32()
        _lib.check(_lib.lib().fse_shard_levels(self.handle, ctypes.byref(n), None))
        self.n_levels = n.value
        fl = np.zeros(max(self.n_levels, 1), dtype=np.int32)
        _lib.check(_lib.lib().fse_shard_levels(self.handle, ctypes.byref(n), _lib.ptr32(fl)))
        self.flags = fl[: self.n_levels]

    def run(self, level: int, level_hi: int | None = None) -> None:
        """Launch levels [level, level_hi) (default: the one level) in one call."""
        hi = level + 1 if level_hi is None else level_hi
        _lib.check(_lib.lib().fse_shard_run(self.handle, level, hi, self.stream))

    def close(self) -> None:
        if self.handle is not None and self.handle.value:
            _lib.check(_lib.lib().fse_shard_close(self.handle, self.stream))
            self.handle = None


class PeerLink:
    """Fused halo exchange over peer memory (C ABI fse_ipc_* / fse_shard_set_peers):
    this rank's frame and a pair of device flags are exported through CUDA IPC,
    the neighbours' are mapped here, and a shard then runs all its levels in
    one call -- the level kernel stores band-edge blocks straight into the
    neighbour's frame and the streams order the levels through the flags (no
    NCCL on the data path, no host round trip per level).  Construct once per
    frame buffer on every rank (collective: all_gather of the handles)."""

    def __init__(self, image_dev, rank: int, world: int, dist, group=None):
        L = _lib.lib()
        self.rank, self.world = rank, world
        self.flags = None
        mine = None
        try:  # the handle exchange below is collective: always reach it
            fl = ctypes.c_void_p()
            _lib.check(L.fse_flags_alloc(ctypes.byref(fl)))
            self.flags = fl
            h_img = ctypes.create_string_buffer(_lib.FSE_IPC_HANDLE_BYTES)
            h_flg = ctypes.create_string_buffer(_lib.FSE_IPC_HANDLE_BYTES)
            _lib.check(L.fse_ipc_handle(ctypes.c_void_p(image_dev.data_ptr()), h_img))
            _lib.check(L.fse_ipc_handle(fl, h_flg))
            mine = (bytes(h_img.raw), bytes(h_flg.raw))
        except Exception:
            mine = None
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        if any(h is None for h in allh):
            self._opened = []
            self.close()
            raise RuntimeError("peer mapping unavailable on some rank")
        self._opened = []

        def open_(h):
            ptr = ctypes.c_void_p()
            _lib.check(L.fse_ipc_open(ctypes.create_string_buffer(h, len(h)), ctypes.byref(ptr)))
            self._opened.append(ptr)
            return ptr

        try:
            self.up = (open_(allh[rank - 1][0]), open_(allh[rank - 1][1])) if rank > 0 else (None, None)
            self.down = (open_(allh[rank + 1][0]), open_(allh[rank + 1][1])) if rank < world - 1 else (None, None)
        except Exception:
            self.close()
            raise
        # flag values of successive runs: [base, base + n_levels], each run's
        # base above the previous run's last value (flags start at 0), so a
        # run with fewer levels than the last one never sees stale values
        self.next_base = 1

    def attach(self, executor) -> int:
        """Route this shard's halos through peer memory for its next run.
        Returns the C status (FSE_ENOTSUP when the shard cannot fuse the
        exchange) instead of raising, so the ranks can agree on a fallback."""
        rc = _lib.lib().fse_shard_set_peers(executor.handle, self.up[0], self.up[1], self.down[0],
                                            self.down[1], self.flags, self.next_base)
        if rc == 0:
            self.next_base += executor.n_levels + 1
        return rc

    @staticmethod
    def detach(executor) -> None:
        _lib.check(_lib.lib().fse_shard_set_peers(executor.handle, None, None, None, None, None, 0))

    def close(self) -> None:
        L = _lib.lib()
        for p in self._opened:
            L.fse_ipc_close(p)
        self._opened = []
        if self.flags is not None:
            L.fse_flags_free(self.flags)
            self.flags = None


def open_peer_link(image_dev, rank: int, world: int, dist, group=None):
    """PeerLink on every rank, or None on every rank when any rank cannot map
    its neighbours (no peer access between the devices, no IPC): the ranks
    agree through one all_gather, and the caller falls back to the collective
    exchange."""
    link, ok = None, True
    try:
        link = PeerLink(image_dev, rank, world, dist, group)
    except Exception:  # mapping failed on this rank
        ok = False
    flags = [None] * world
    dist.all_gather_object(flags, ok, group=group)
    if all(flags):
        return link
    if link is not None:
        link.close()
    return None


def attach_all(executor, link: PeerLink, dist, group=None) -> bool:
    """Attach every rank's shard to its peers, or none: the fused exchange
    needs the fast kernel on every rank (fse_shard_set_peers answers
    FSE_ENOTSUP otherwise, e.g. fft_size=None or a window too large for the
    fp64 F = 128 half plane), so the
    ranks agree through one all_gather and fall back to the collective
    exchange together."""
    rc = link.attach(executor)
    if rc not in (0, _lib.FSE_ENOTSUP):
        _lib.check(rc)
    oks = [None] * link.world
    dist.all_gather_object(oks, rc == 0, group=group)
    if all(oks):
        return True
    if rc == 0:
        PeerLink.detach(executor)
    return False


def run_levels_p2p(executor, link: PeerLink, dist=None, group=None) -> bool:
    """The whole level sequence of one shard with the fused exchange.  With
    `dist`, the ranks first agree (attach_all); returns False, having run
    nothing, when some rank's shard cannot fuse the exchange."""
    if dist is not None:
        if not attach_all(executor, link, dist, group):
            return False
    else:
        _lib.check(link.attach(executor))
    _lib.check(_lib.lib().fse_shard_run(executor.handle, 0, executor.n_levels, executor.stream))
    return True


def run_levels_collective(executor, image_dev, rank, world, bands, R, B, H, dist, group=None) -> int:
    """The per-level send/recv protocol (run_levels) with the edge flags of
    every rank gathered first."""
    import torch

    flags_all = [executor.flags]
    if world > 1:
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.as_tensor(executor.flags, dtype=torch.int32, device=dev)
        gathered = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gathered, t, group=group)
        flags_all = [g.cpu().numpy() for g in gathered]
    return run_levels(executor, image_dev, rank, world, bands, flags_all, executor.n_levels, R, B, H, dist,
                      group)


def conceal_strips(image, mask, params: FseParams, precision: str = "fp64", order: str = "optimized",
                   group=None, gather: bool = True, transport: str = "p2p", plan_on: str = "rank0"):
    """Conceal one frame on all ranks of the default process group (one GPU per
    rank).  Returns (image, mask) numpy arrays on rank 0 when gather=True (other
    ranks get None), else this rank's band rows and its band.  plan_on "rank0"
    = rank 0 plans the frame and broadcasts the plan (broadcast_plan), "all" =
    every rank plans it (deterministic, identical).  transport "p2p"
    = fused halo exchange over peer memory (PeerLink), "collective" = per-level
    send/recv over torch.distributed (NCCL on GPUs)."""
    if transport not in ("p2p", "collective"):
        raise ValueError("transport must be 'p2p' or 'collective'")
    if plan_on not in ("rank0", "all"):
        raise ValueError("plan_on must be 'rank0' (plan once, broadcast) or 'all' (every rank plans)")
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    H, W = mask.shape
    if world > 1 and plan_on == "rank0":
        hg = host_group(dist, group)
        src = 0 if group is None else dist.get_global_rank(group, 0)
        plan = broadcast_plan(mask, params, order, rank, dist, hg, src, precision=precision)
    else:
        plan = build_plan(mask, params, order)
        balance_for_device(plan, params, precision)
    B = params.block_size
    R = halo_rows(params)
    processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(plan.rows, plan.cols)
    bands = band_partition(processed.sum(axis=1), world, R)
    tdt = torch.float32 if precision == "fp32" else torch.float64
    img_d = torch.as_tensor(np.ascontiguousarray(image)).to(device="cuda", dtype=tdt)
    msk_d = torch.from_numpy(mask).cuda()
    out_d = torch.empty_like(msk_d)
    ex = ShardExecutor(plan, bands[rank], img_d, msk_d, out_d, params, precision)
    link = open_peer_link(img_d, rank, world, dist, group) if world > 1 and transport == "p2p" else None
    fused = False
    if link is not None:
        try:
            fused = run_levels_p2p(ex, link, dist, group)
            if fused:
                ex.close()
                torch.cuda.synchronize()
                dist.barrier(group=group)  # every rank's peer stores have landed
        finally:
            link.close()
    if not fused:
        run_levels_collective(ex, img_d, rank, world, bands, R, B, H, dist, group)
        ex.close()
    lo, hi = bands[rank]
    y0, y1 = lo * B, min(H, hi * B)
    if not gather:
        return img_d[y0:y1].double().cpu().numpy(), out_d[y0:y1].cpu().numpy(), bands[rank]
    if world > 1:
        host = dist.get_backend(group) == "gloo"  # gloo moves host memory only
        if rank == 0:
            for r in range(1, world):
                a, b = bands[r][0] * B, min(H, bands[r][1] * B)
                for t in (img_d[a:b], out_d[a:b]):
                    if host:
                        hb = t.cpu()
                        dist.recv(hb, r, group)
                        t.copy_(hb)
                    else:
                        dist.recv(t, r, group)
        else:
            for t in (img_d[y0:y1].contiguous(), out_d[y0:y1].contiguous()):
                dist.send(t.cpu() if host else t, 0, group)
    if rank != 0:
        return None
    return img_d.double().cpu().numpy(), out_d.cpu().numpy()
