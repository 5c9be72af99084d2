"""Dev: per-config device timing of the level pipeline (plans prebuilt)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth

CASES = [
    (1, 4, 64, 100, "optimized", "fp64"),
    (2, 4, 64, 100, "optimized", "fp32"), (2, 4, 64, 100, "optimized", "fp64"),
    (2, 4, 64, 100, "linescan", "fp32"), (2, 4, 64, 100, "linescan", "fp64"),
    (3, 4, 64, 200, "optimized", "fp32"),
    (5, 2, 32, 100, "optimized", "fp32"), (5, 4, 64, 100, "optimized", "fp32"),
    (5, 8, 128, 100, "optimized", "fp32"),
]
only = sys.argv[1:]
for cfg, B, F, I, order, prec in CASES:
    if only and str(cfg) not in only:
        continue
    img, mask = synth.config_scene(cfg)
    p = P.FseParams(d=14, iterations=I, block_size=B, fft_size=F)
    t = time.perf_counter()
    plan = P.build_plan(mask, p, order)
    tp = time.perf_counter() - t
    tdt = torch.float32 if prec == "fp32" else torch.float64
    src = torch.from_numpy(img).cuda().to(tdt)
    work = torch.empty_like(src)
    m = torch.from_numpy(mask).cuda()
    mo = torch.empty_like(m)
    def run():
        work.copy_(src)
        P.run_frames_device([plan], [work], [m], [mo], p, prec)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 3
    e0.record()
    for _ in range(reps):
        run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 17.0 * I * F * (F // 2 + 1) * plan.n_processed
    print(f"cfg{cfg} B={B} F={F} I={I} {order:9s} {prec}: blocks {plan.n_processed} levels {plan.n_levels} "
          f"batches {plan.n_batches} plan {tp*1e3:.0f} ms  device {ms:.1f} ms  "
          f"{plan.n_processed/ms*1e3:.0f} blocks/s  {flops/ms/1e9:.2f} TFLOP/s", flush=True)
