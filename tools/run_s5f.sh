# check of the adopted build: GPU tests, smoke, configs 1-4
set -x
mkdir -p gpurun_out
T=${TAG:-s5f}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
python tools/variant_smoke.py > gpurun_out/${T}_variants.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_variants.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c4.json 2>gpurun_out/${T}_c4.err
for c in 1 2 3; do
  st=10; [ $c = 3 ] && st=3
  python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_c${c}.json 2>&1
done
tail -n 3 gpurun_out/${T}_tests.log gpurun_out/${T}_smoke.log gpurun_out/${T}_variants.log
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5f")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), runs)
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
