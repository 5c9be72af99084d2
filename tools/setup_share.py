"""Dev: kernel time vs iteration count on config-4 frames (setup share = time at I=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth, _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
sc = [synth.config_scene(4, f) for f in range(n)]
imgs = torch.from_numpy(np.stack([s[0] for s in sc])).cuda()
msks = torch.from_numpy(np.stack([s[1] for s in sc])).cuda()
L = _lib.lib()
for I in (1, 2, 10, 50, 100):
    p = P.FseParams(d=14, iterations=I, block_size=4, fft_size=64)
    plans = P.build_plans(list(msks.cpu().numpy()), p)
    work = torch.empty(imgs.shape, dtype=torch.float32 if prec == "fp32" else torch.float64, device="cuda")
    out = torch.empty_like(msks)
    for rep in range(3):
        work.copy_(imgs)
        torch.cuda.synchronize()
        L.fse_timing_read(None, None, None)
        L.fse_timing_enable(1)
        P.run_frames_device(plans, list(work), list(msks), list(out), p, prec)
        torch.cuda.synchronize()
        L.fse_timing_enable(0)
        kms = ctypes.c_double()
        L.fse_timing_read(ctypes.byref(kms), None, None)
    blocks = sum(pl.n_processed for pl in plans)
    print(f"I={I:3d}: kernel {kms.value:8.2f} ms  {1e3 * kms.value / blocks:7.3f} us/block")
