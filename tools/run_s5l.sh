# level balancing (narrow tail levels filled with slack blocks of the wide levels): A/B + GPU tests
mkdir -p gpurun_out
T=${TAG:-s5l}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
for bal in 0 1; do
  for c in 1 2 3; do
    st=10; [ $c = 3 ] && st=3
    FSE_BALANCE=$bal python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bal${bal}_c$c.json 2>&1
  done
  FSE_BALANCE=$bal python bench.py --config 3 --precision fp32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bal${bal}_c3f32.json 2>&1
  FSE_BALANCE=$bal python bench.py --config 3 --defaults --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bal${bal}_c3def.json 2>&1
  for B in 2 4 8; do FSE_BALANCE=$bal python bench.py --config 5 --block $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bal${bal}_c5b$B.json 2>&1; done
done
FSE_BALANCE_WAVE=1 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_wave_c3.json 2>&1
FSE_BALANCE_WAVE=1 python bench.py --config 5 --block 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_wave_c5b4.json 2>&1
tail -n 3 gpurun_out/${T}_tests.log
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5l")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        runs={k:round(v["ms"],2) for k,v in (d.get("runs") or {}).items() if isinstance(v,dict) and "ms" in v}
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), "e2e", round((d.get("e2e") or {}).get("ms_per_step") or 0,2), runs)
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-400:])
PY
