"""Dev driver for ncu / diagnostics: conceal N config-4 frames (twice)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth, _lib

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=8)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--guard", default="off")
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--block", type=int, default=4)
ap.add_argument("--fft", type=int, default=64)
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--stats", action="store_true", help="fp32 vs fp64 deviation statistics")
a = ap.parse_args()
L = _lib.lib()
t0, t1 = (-1.0, 0.0) if a.guard == "off" else (float(x) for x in a.guard.split(","))
L.fse_set_guard(t0, t1)
sc = [synth.config_scene(a.config, f) for f in range(a.frames)]
imgs = np.stack([s[0] for s in sc]); msks = np.stack([s[1] for s in sc])
p = P.FseParams(d=14, iterations=a.iters, block_size=a.block, fft_size=a.fft)
import torch
tdt = torch.float32 if a.precision == "fp32" else torch.float64
img_d = torch.from_numpy(imgs).cuda().to(tdt)
msk_d = torch.from_numpy(msks).cuda()
out_d = torch.empty_like(msk_d)
plans = P.build_plans(list(msks), p)
for _ in range(a.reps):  # one call, every level of all frames merged (no chunking)
    work = img_d.clone()
    P.run_frames_device(plans, list(work), list(msk_d), list(out_d), p, a.precision)
torch.cuda.synchronize()
out = work.cpu().numpy()
if a.stats:
    o64, _, _ = P.conceal_batch(imgs, msks, p, precision="fp64", reports=False)
    lost = msks == 1
    d = np.abs(out.astype(np.float64) - o64)[lost]
    def psnr(x):
        mse = np.mean((x[lost] - imgs[lost].astype(np.float64)) ** 2)
        return 10 * np.log10(255 ** 2 / mse)
    print(f"{a.precision} guard={a.guard}: max|d| {d.max():.3f}  frac>0.5 {(d > 0.5).mean():.2e}  "
          f"n>0.5 {(d > 0.5).sum()}  psnr {psnr(out.astype(np.float64)):.4f} vs fp64 {psnr(o64):.4f}")
print("done")
