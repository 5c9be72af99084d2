"""Dev diagnostic: fp32 path vs the reference (golden) / fp64 path."""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [R, os.path.join(R, "tests")]
import numpy as np
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
from helpers import conceal_case

def psnr(orig, res, mask):
    region = mask != 0
    mse = float(np.mean((orig[region] - res[region]) ** 2))
    return 10 * np.log10(255.0 ** 2 / mse)

g = np.load(os.path.join(R, "tests/golden/conceal_cases.npz"))
for i in [2, 3, 4, 5, 6, 7]:
    c = conceal_case(g, i)
    p = P.FseParams(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"], iterations=c["iterations"],
                    block_size=c["block_size"], fft_size=c["fft"])
    out, _, _ = P.conceal(c["image"], c["mask"], p, c["order"], precision="fp32")
    lost = c["mask"] == 1
    d = np.abs(out - c["out_image"])[lost]
    t = c["image"].astype(np.float64)
    print(f"case {i} {c['name']}: max {d.max():.3g} frac>0.5 {(d>0.5).mean():.4f} "
          f"dpsnr {psnr(t, out, c['mask']) - psnr(t, c['out_image'], c['mask']):+.4f} (ref {psnr(t, c['out_image'], c['mask']):.2f} dB)")
f = np.load(os.path.join(R, "tests/golden/full_cfg.npz"))
for k in range(3):
    img, mask = synth.config_scene(int(f[f"f{k}_config"]))
    p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
    out, _, _ = P.conceal(img, mask, p, str(f[f"f{k}_order"]), precision="fp32")
    lost = mask == 1
    ref = img.astype(np.float64).copy(); ref[lost] = f[f"f{k}_lost_values"]
    d = np.abs(out - ref)[lost]
    t = img.astype(np.float64)
    print(f"full cfg{int(f[f'f{k}_config'])} {str(f[f'f{k}_order'])}: max {d.max():.3g} frac>0.5 {(d>0.5).mean():.4f} "
          f"dpsnr {psnr(t, out, mask) - psnr(t, ref, mask):+.4f} (ref {psnr(t, ref, mask):.2f} dB)")
for cfg, it in [(3, 200), (4, 100)]:
    img, mask = synth.config_scene(cfg)
    p = P.FseParams(d=14, iterations=it, block_size=4, fft_size=64)
    o32, _, _ = P.conceal(img, mask, p, precision="fp32")
    o64, _, _ = P.conceal(img, mask, p, precision="fp64")
    lost = mask == 1
    d = np.abs(o32 - o64)[lost]
    t = img.astype(np.float64)
    print(f"cfg{cfg} fp32 vs fp64: max {d.max():.3g} frac>0.5 {(d>0.5).mean():.4f} dpsnr {psnr(t, o32, mask) - psnr(t, o64, mask):+.4f} (fp64 {psnr(t, o64, mask):.2f} dB)")
