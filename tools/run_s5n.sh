# level balancing modes: narrow fill (default) / + levels below one wave up to the wave (1) / every level up to a wave (2)
mkdir -p gpurun_out
T=${TAG:-s5n}
for mode in 0 1 2; do
  FSE_BALANCE_WAVE=$mode python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_m${mode}_c3.json 2>&1
  FSE_BALANCE_WAVE=$mode python bench.py --config 3 --precision fp32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_m${mode}_c3f32.json 2>&1
  FSE_BALANCE_WAVE=$mode python bench.py --config 3 --defaults --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_m${mode}_c3def.json 2>&1
  for B in 4 8; do FSE_BALANCE_WAVE=$mode python bench.py --config 5 --block $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_m${mode}_c5b$B.json 2>&1; done
done
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5n")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1))
    except Exception as e:
        print(f.split("/")[-1], "ERR", open(f).read()[-300:])
PY
