mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
python tools/bench_configs.py 2 3 5 > gpurun_out/t_cfg.txt 2>&1
FSE_TRACK_BELOW=0 python tools/bench_configs.py 3 > gpurun_out/t_cfg_lazy.txt 2>&1
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-second > gpurun_out/t_bench.json 2>&1
python - <<'PY' > gpurun_out/t_same.txt 2>&1
# tracked and lazy argmax give bit-identical frames
import os, numpy as np, torch, ctypes
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
img, mask = synth.config_scene(3)
p = P.FseParams(d=14, iterations=200, block_size=4, fft_size=64)
plan = P.build_plan(mask, p)
outs = []
for below in ("100000000", "0"):
    os.environ["FSE_TRACK_BELOW"] = below
import subprocess, sys
PY
for b in 100000000 0; do FSE_TRACK_BELOW=$b python - <<'PY' >> gpurun_out/t_same.txt 2>&1
import numpy as np, torch, hashlib
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
img, mask = synth.config_scene(3)
p = P.FseParams(d=14, iterations=200, block_size=4, fft_size=64)
o, m, _ = P.conceal_batch(img[None], mask[None], p, precision="fp32", reports=False)
print(hashlib.sha1(o.tobytes()).hexdigest(), hashlib.sha1(m.tobytes()).hexdigest())
PY
done
