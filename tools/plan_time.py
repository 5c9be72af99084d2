import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_00233_b200 import synth, _lib
lib = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".so") else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2207_00233_b200", "libfse_b200.so"))
img, mask = synth.config_scene(5)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
F = {2: 32, 4: 64, 8: 128}[B]
pc = _lib.FseParamsC(14, B, 100, F, F, 0.8, 0.2, 0.5)
m = np.ascontiguousarray(mask)
h = ctypes.c_void_p()
lib.fse_plan_build.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
for i in range(int(os.environ.get("REPS", 2))):
    t = time.perf_counter()
    rc = lib.fse_plan_build(m.ctypes.data, m.shape[0], m.shape[1], ctypes.byref(pc), 0, ctypes.byref(h))
    print("rc", rc, f"{1e3*(time.perf_counter()-t):.1f} ms", flush=True)
    lib.fse_plan_free(h)
