"""Dev/test driver: conceal one frame strip-sharded over `world` processes on
the visible GPU(s) (gloo for the host-side collectives), with the fused
peer-memory halo exchange and with the collective one; rank 0 compares both
with a whole-frame run.  usage: python tests/strips_p2p_driver.py [world] [config] [B]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def worker(rank, world, port, cfg, B, crop, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2207_00233_b200 as P
    from paper_2207_00233_b200 import strips, synth
    img, mask = synth.config_scene(cfg)
    if crop:
        img, mask = img[:crop[0], :crop[1]].copy(), mask[:crop[0], :crop[1]].copy()
    F = {2: 32, 4: 64, 8: 128}[B]
    p = P.FseParams(d=14, iterations=40, block_size=B, fft_size=F)
    res = {}
    for tr, prec in (("p2p", "fp32"), ("collective", "fp32"), ("p2p", "fp32"), ("p2p", "fp64")):
        t = time.perf_counter()
        out = strips.conceal_strips(img, mask, p, prec, transport=tr)
        res.setdefault((tr, prec), []).append((out, time.perf_counter() - t))
    # one PeerLink reused over runs whose level counts shrink (flag bases must
    # keep increasing: ADVICE r1), frame buffer fixed as in bench.py
    H, W = mask.shape
    work = torch.empty((H, W), dtype=torch.float64, device="cuda")
    msk = torch.from_numpy(mask).cuda()
    mout = torch.empty_like(msk)
    link = strips.open_peer_link(work, rank, world, dist)
    R = strips.halo_rows(p)
    reuse = []
    masks = [mask]
    m2 = mask.copy()
    m2[:, W // 2:] = 0  # half the losses: fewer levels
    masks.append(m2)
    for mk in masks + masks[:1]:
        plan = P.build_plan(mk, p)
        processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(plan.rows, plan.cols)
        bands = strips.band_partition(processed.sum(axis=1), world, R)
        work.copy_(torch.from_numpy(img.astype(np.float64)))
        msk.copy_(torch.from_numpy(mk))
        ex = strips.ShardExecutor(plan, bands[rank], work, msk, mout, p, "fp64")
        fused = link is not None and strips.run_levels_p2p(ex, link, dist)
        if not fused:
            strips.run_levels_collective(ex, work, rank, world, bands, R, B, H, dist)
        ex.close()
        torch.cuda.synchronize()
        dist.barrier()
        lo, hi = bands[rank]
        y0, y1 = lo * B, min(H, hi * B)
        rows = work[y0:y1].cpu()
        gathered = [None] * world
        dist.all_gather_object(gathered, (y0, y1, rows.numpy()))
        full = np.zeros((H, W))
        for a0, a1, r in gathered:
            full[a0:a1] = r
        reuse.append((mk, full, fused, plan.n_levels))
    if link is not None:
        link.close()
    # default FseParams DFT size (fft_size=None): the fused exchange is not
    # available, every rank must fall back to the collective one together
    pn = P.FseParams(d=14, iterations=20, block_size=B)
    outn = strips.conceal_strips(img, mask, pn, "fp64", transport="p2p")
    if rank == 0:
        ok = {}
        for prec in ("fp32", "fp64"):
            whole, wm, _ = P.conceal(img, mask, p, precision=prec)
            for (tr, pr), runs in res.items():
                if pr == prec:
                    ok[f"{tr}-{pr}"] = all(np.array_equal(o[0], whole) and np.array_equal(o[1], wm) for o, _ in runs)
        for i, (mk, full, fused, nl) in enumerate(reuse):
            whole, _, _ = P.conceal(img, mk, p, precision="fp64")
            ok[f"reuse{i}-fused{int(fused)}-levels{nl}"] = bool(np.array_equal(full, whole)) and (
                fused or link is None)
        wn, wnm, _ = P.conceal(img, mask, pn, precision="fp64")
        ok["fft_none_fallback"] = bool(np.array_equal(outn[0], wn) and np.array_equal(outn[1], wnm))
        q.put(ok)
    dist.barrier()
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    crop = (256, 384) if cfg == 5 else None
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29000 + os.getpid() % 1000
    ps = [ctx.Process(target=worker, args=(r, world, port, cfg, B, crop, q)) for r in range(world)]
    for p in ps:
        p.start()
    deadline = time.time() + 240
    for p in ps:
        p.join(max(1, deadline - time.time()))
    hung = [p for p in ps if p.is_alive()]
    for p in hung:
        p.kill()
    if hung:
        print("TIMEOUT")
        sys.exit(3)
    ok = q.get() if not q.empty() else None
    print("result", ok)
    sys.exit(0 if ok and all(ok.values()) else 1)


if __name__ == "__main__":
    main()
