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
    if rank == 0:
        ok = {}
        for prec in ("fp32", "fp64"):
            whole, wm, _ = P.conceal(img, mask, p, precision=prec)
            for (tr, pr), runs in res.items():
                if pr == prec:
                    ok[f"{tr}-{pr}"] = all(np.array_equal(o[0], whole) and np.array_equal(o[1], wm) for o, _ in runs)
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
