# A/B in one call: the previous commit's tree (ab_base/) against this tree with the cache off / on
set -x
mkdir -p gpurun_out
T=${TAG:-s4d}
ROOT=$PWD
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second"
for rep in 1 2; do
  (cd ab_base && $B > $ROOT/gpurun_out/${T}_base_$rep.json 2> $ROOT/gpurun_out/${T}_base_$rep.err)
  FSE_WCACHE=0 $B > gpurun_out/${T}_wc0_$rep.json 2> gpurun_out/${T}_wc0_$rep.err
  FSE_WCACHE=1 $B > gpurun_out/${T}_wc1_$rep.json 2> gpurun_out/${T}_wc1_$rep.err
done
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s4d")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["dtype"], round(d["ms_per_step"],1), round(d["kernel_ms_per_step"],1), round(d["roofline"]["frac"],4), "enq", round(d["host_enqueue_ms_per_step"],1))
    except Exception as e:
        print(f, "ERR", e); print(open(f.replace(".json",".err")).read()[-1500:])
PY
