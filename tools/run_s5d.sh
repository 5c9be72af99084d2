# config 4 fp64 (cached-W kernel): frame groups 1/2/3/4/6 re-measured
set -x
mkdir -p gpurun_out
T=${TAG:-s5d}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second"
for g in 2 1 3 4 6 2; do
  FSE_GROUPS=$g $B > gpurun_out/${T}_g$g.json 2>gpurun_out/${T}_g$g.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/${T}_g$g.json").read().strip().splitlines()[-1])
print("groups $g", round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), d.get("gpu_launches"))
PY
done
