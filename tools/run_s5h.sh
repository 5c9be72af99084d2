# which host call stalls a device-resident step: FSE_OPEN_TIMING trace of 5 bench runs
mkdir -p gpurun_out
T=${TAG:-s5h}
for i in 1 2 3 4 5; do
  FSE_OPEN_TIMING=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_$i.json 2>gpurun_out/${T}_$i.err
done
nproc; uptime
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5h")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split("/")[-1], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), d.get("host_enqueue_ms_steps"))
PY
