import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [R, os.path.join(R, "tests")]
import numpy as np
import paper_2207_00233_b200 as P
from helpers import conceal_case
g = np.load(os.path.join(R, "tests/golden/conceal_cases.npz"))
c = conceal_case(g, int(sys.argv[1]))
prec = sys.argv[2]
its = int(sys.argv[3]) if len(sys.argv) > 3 else c["iterations"]
p = P.FseParams(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"], iterations=its,
                block_size=c["block_size"], fft_size=c["fft"])
img, msk, rep = P.conceal(c["image"], c["mask"], p, c["order"], precision=prec)
print("ok", sys.argv[1:], os.environ.get("FSE_CLUSTER"), np.abs(img - c["out_image"]).max())
print("nan samples", int(np.isnan(img).sum()), "inf", int(np.isinf(img).sum()))
