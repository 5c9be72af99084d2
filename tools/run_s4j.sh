# (1) previous tree vs this tree (cache off / on), (2) cluster variants on the latency-bound configs (fp64)
set -x
mkdir -p gpurun_out
T=${TAG:-s4j}
ROOT=$PWD
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second"
(cd ab_base && $B > $ROOT/gpurun_out/${T}_base.json 2> $ROOT/gpurun_out/${T}_base.err)
FSE_WCACHE=0 $B > gpurun_out/${T}_wc0.json 2> gpurun_out/${T}_wc0.err
FSE_WCACHE=1 $B > gpurun_out/${T}_wc1.json 2> gpurun_out/${T}_wc1.err
for v in main cl cl12; do
  for cm in 2 4; do
    if [ $v = main ] && [ $cm = 4 ]; then continue; fi
    lib=""; [ $v != main ] && lib=$PWD/paper_2207_00233_b200/variants/libfse_b200_$v.so
    for c in 1 2; do
      FSE_LIB=$lib FSE_CLUSTER=$cm python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c${c}_${v}_cm$cm.json 2>&1
    done
  done
done
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s4j")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), runs)
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
