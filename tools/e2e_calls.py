"""Dev: wall time of consecutive conceal_batch calls (config 4, 64 frames, pinned)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
from concurrent.futures import ThreadPoolExecutor

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
with ThreadPoolExecutor(16) as ex:
    sc = list(ex.map(lambda f: synth.config_scene(4, f), range(n)))
imgs_h = torch.from_numpy(np.stack([s[0] for s in sc])).pin_memory()
msks_h = torch.from_numpy(np.stack([s[1] for s in sc])).pin_memory()
p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
oi = torch.empty(imgs_h.shape, dtype=torch.float32, pin_memory=True)
om = torch.empty(msks_h.shape, dtype=torch.uint8, pin_memory=True)
import gc
if os.environ.get("GC_MODE") == "freeze":
    gc.collect(); gc.freeze()
elif os.environ.get("GC_MODE") == "off":
    gc.disable()
if os.environ.get("GC_LOG"):
    gc.callbacks.append(lambda phase, info: print(f"gc {phase} gen{info['generation']} {time.perf_counter():.4f}", flush=True) if info['generation'] == 2 else None)
for i in range(int(os.environ.get("CALLS", 8))):
    t = time.perf_counter()
    P.conceal_batch(imgs_h, msks_h, p, out_images=oi, out_masks=om, reports=False)
    print(f"call {i}: {1e3 * (time.perf_counter() - t):.1f} ms")
