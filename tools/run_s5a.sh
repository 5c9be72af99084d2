# A/B on one box: the r2y tree (ab_base = ad374c9) vs this tree on the latency-bound configs
set -x
mkdir -p gpurun_out
T=${TAG:-s5a}
ROOT=$PWD
for rep in 1 2; do
for c in 1 2 3; do
  st=10; [ $c = 3 ] && st=3
  (cd ab_base && python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > $ROOT/gpurun_out/${T}_base_c${c}_$rep.json 2>&1)
  python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_head_c${c}_$rep.json 2>&1
  FSE_WCACHE=0 python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_headwc0_c${c}_$rep.json 2>&1
done
done
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5a")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), runs)
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
