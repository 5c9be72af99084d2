# A/B: integer best-of-bins compare (ti), masked wrap offset of the u-a gather (w), both (tw) vs main
set -x
mkdir -p gpurun_out
T=${TAG:-s5e}
V=${VARIANTS:-"main ti w tw"}
for rep in 1 2; do
for v in $V; do
  lib=""; [ $v != main ] && lib=$PWD/paper_2207_00233_b200/variants/libfse_b200_$v.so
  FSE_LIB=$lib python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c4_${v}_$rep.json 2>gpurun_out/${T}_c4_${v}_$rep.err
  for c in 1 2 3; do
    st=10; [ $c = 3 ] && st=3
    FSE_LIB=$lib python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_c${c}_${v}_$rep.json 2>&1
  done
done
done
for v in $V; do
  [ $v = main ] && continue
  FSE_LIB=$PWD/paper_2207_00233_b200/variants/libfse_b200_$v.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_tests_$v.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests_$v.log
done
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5e")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), runs)
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-600:])
PY
for f in gpurun_out/${T}_tests_*.log; do echo $f; tail -n 3 $f; done
