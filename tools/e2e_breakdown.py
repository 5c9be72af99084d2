"""Dev: where the e2e time of conceal_batch goes (config 4, 64 frames)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
from concurrent.futures import ThreadPoolExecutor
with ThreadPoolExecutor(16) as ex:
    sc = list(ex.map(lambda f: synth.config_scene(4, f), range(64)))
imgs_h = torch.from_numpy(np.stack([s[0] for s in sc])).pin_memory()
msks_h = torch.from_numpy(np.stack([s[1] for s in sc])).pin_memory()
p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
oi = torch.empty(imgs_h.shape, dtype=torch.float32, pin_memory=True)
om = torch.empty(msks_h.shape, dtype=torch.uint8, pin_memory=True)
for _ in range(2):
    P.conceal_batch(imgs_h, msks_h, p, out_images=oi, out_masks=om, reports=False)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
t = [0.0] * 6
t[0] = time.perf_counter(); ev[0].record()
img_d = imgs_h.to("cuda", non_blocking=True).to(torch.float32)
msk_d = msks_h.to("cuda", non_blocking=True)
out_d = torch.empty_like(msk_d)
ev[1].record(); t[1] = time.perf_counter()
plans = P.plan_and_run(list(msks_h.numpy()), list(img_d), list(msk_d), list(out_d), p, "fp32")
ev[2].record(); t[2] = time.perf_counter()
oi.copy_(img_d, non_blocking=True); om.copy_(out_d, non_blocking=True)
ev[3].record(); t[3] = time.perf_counter()
torch.cuda.synchronize(); t[4] = time.perf_counter()
print("device ms: upload %.1f  compute %.1f  download %.1f" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])))
print("host ms: upload-enqueue %.1f  plan+enqueue %.1f  dl-enqueue %.1f  wait %.1f total %.1f" % (1e3*(t[1]-t[0]), 1e3*(t[2]-t[1]), 1e3*(t[3]-t[2]), 1e3*(t[4]-t[3]), 1e3*(t[4]-t[0])))
