# config 4 fp64: a plane for every class map (no computing path in the level kernels) vs the default (maps seen >= 2 times)
set -x
mkdir -p gpurun_out
T=${TAG:-s5c}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second"
$B > gpurun_out/${T}_dflt.json 2>gpurun_out/${T}_dflt.err
FSE_WCACHE_MIN=1 FSE_WCACHE_PLANES=400000 FSE_WCACHE_MB=16384 $B > gpurun_out/${T}_min1.json 2>gpurun_out/${T}_min1.err
FSE_WCACHE_PLANES=400000 FSE_WCACHE_MB=16384 $B > gpurun_out/${T}_min2_big.json 2>gpurun_out/${T}_min2_big.err
$B > gpurun_out/${T}_dflt2.json 2>gpurun_out/${T}_dflt2.err
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5c")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), d.get("weight_spectrum_cache"))
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
