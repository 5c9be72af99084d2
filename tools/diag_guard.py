"""Dev diagnostic: fp32 guard behaviour on golden case 2 (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import _lib
from helpers import conceal_case
g = np.load("tests/golden/conceal_cases.npz")
c = conceal_case(g, 2)
p = P.FseParams(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"], iterations=c["iterations"],
                block_size=c["block_size"], fft_size=c["fft"])
L = _lib.lib()
for tau0, tau1 in [(2e-5, 3e-6), (1.0, 0.0), (-1.0, 0.0), (1e-3, 0.0)]:
    L.fse_set_guard(tau0, tau1)
    L.fse_guard_redo_count(1)
    L.fse_timing_enable(1)
    img, msk, rep, picks = P.conceal(c["image"], c["mask"], p, c["order"], precision="fp32", return_picks=True)
    L.fse_timing_enable(0)
    L.fse_timing_read(None, None, None)
    n = L.fse_guard_redo_count(1)
    err = np.abs(img - c["out_image"])
    print(f"tau0={tau0} tau1={tau1}: redo={n} max err {err.max():.3e} n>0.5 {(err > 0.5).sum()}")
img64, _, _, picks64 = P.conceal(c["image"], c["mask"], p, c["order"], precision="fp64", return_picks=True)
print("fp64 max err", np.abs(img64 - c["out_image"]).max())
