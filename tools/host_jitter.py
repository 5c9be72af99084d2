"""Dev: host scheduling jitter on the GPU box: largest gaps in a tight loop
(alone, and while the GPU runs conceal_batch calls in another thread)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def spin(seconds):
    gaps = []
    t_end = time.perf_counter() + seconds
    last = time.perf_counter()
    while last < t_end:
        now = time.perf_counter()
        if now - last > 0.002:
            gaps.append(now - last)
        last = now
    return sorted(gaps)[-5:]


print("alone, 5 s: largest gaps (ms)", [round(1e3 * g, 1) for g in spin(5.0)], flush=True)
import numpy as np
import torch
x = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
def gpu_sync_loop(n):
    for _ in range(n):
        x.add_(1)
        t = time.perf_counter()
        torch.cuda.synchronize()
        d = time.perf_counter() - t
        if d > 0.05:
            print(f"slow synchronize {1e3*d:.1f} ms", flush=True)
t = time.perf_counter(); gpu_sync_loop(2000); print(f"2000 add+sync in {time.perf_counter()-t:.2f} s")
os.system("cat /proc/loadavg; nproc")
