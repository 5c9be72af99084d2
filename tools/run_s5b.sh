# weight-spectrum cache gate by average level width: configs 2, 3, 5 with the gate (default) and forced on (WIDTH=0)
set -x
mkdir -p gpurun_out
T=${TAG:-s5b}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
FSE_WCACHE_ENTRIES=1 FSE_WCACHE_WIDTH=0 timeout 1000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests_forced.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests_forced.log
for c in 2 3; do
  st=10; [ $c = 3 ] && st=3
  python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_gate_c${c}.json 2>&1
  FSE_WCACHE_WIDTH=0 python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_w0_c${c}.json 2>&1
done
for B in 4 8; do
  python bench.py --config 5 --block $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_gate_c5b$B.json 2>&1
  FSE_WCACHE_WIDTH=0 python bench.py --config 5 --block $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_w0_c5b$B.json 2>&1
done
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_gate_c4.json 2>&1
tail -2 gpurun_out/${T}_tests.log gpurun_out/${T}_tests_forced.log
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5b")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), runs)
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
