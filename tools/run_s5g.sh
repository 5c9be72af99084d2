# step-time stability of the default bench line with the loop-mode clock sampler (3 runs), plus config 1
mkdir -p gpurun_out
T=${TAG:-s5g}
for i in 1 2 3 4; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-second > gpurun_out/${T}_c4_$i.json 2>gpurun_out/${T}_c4_$i.err
done
python bench.py --config 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_c1.json 2>&1
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5g")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), "host", round(d.get("host_enqueue_ms_per_step") or 0,1), "e2e", (d.get("e2e") or {}).get("ms_per_step"), d["clocks"])
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
