"""Host planner scaling: build_plans wall time for config-4 frames vs threads."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
msks = [synth.config_scene(4, f)[1] for f in range(n)]
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for th in (1, 2, 4, 8, 16, 32, 0):
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        pl = P.build_plans(msks, p, "optimized", th)
        ts.append(round((time.perf_counter() - t) * 1e3, 1))
        del pl
    print(f"threads {th:2d}: {ts} ms for {n} frames")
