# latency-bound configs with a cached W for EVERY window (no computing path in the level kernels)
mkdir -p gpurun_out
T=${TAG:-s5j}
run() { # name, env...
  name=$1; shift
  for c in 1 2 3; do
    st=10; [ $c = 3 ] && st=3
    env "$@" python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_${name}_c$c.json 2>&1
  done
  env "$@" python bench.py --config 5 --block 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_${name}_c5b4.json 2>&1
  env "$@" python bench.py --config 5 --block 8 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_${name}_c5b8.json 2>&1
}
run dflt FSE_NOP=1
run min1 FSE_WCACHE_WIDTH=0 FSE_WCACHE_ENTRIES=1 FSE_WCACHE_MIN=1 FSE_WCACHE_PLANES=400000 FSE_WCACHE_MB=16384
run min2 FSE_WCACHE_WIDTH=0 FSE_WCACHE_ENTRIES=1
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5j")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), runs, d.get("weight_spectrum_cache"))
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-400:])
PY
