# first chunk on a side stream (its narrow tail overlaps the rest's wide head): A/B on the default bench line + GPU tests
mkdir -p gpurun_out
T=${TAG:-s5o}
for rep in 1 2; do for ov in 0 1; do
  FSE_OVERLAP_CHUNKS=$ov python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_ov${ov}_$rep.json 2>gpurun_out/${T}_ov${ov}_$rep.err
done; done
FSE_OVERLAP_CHUNKS=1 python bench.py --precision fp32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_ov1_f32.json 2>&1
FSE_OVERLAP_CHUNKS=0 python bench.py --precision fp32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_ov0_f32.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -n 3 gpurun_out/${T}_tests.log
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s5o")
for f in sorted(glob.glob(f"gpurun_out/{T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["dtype"], round(d["ms_per_step"],2), round(d.get("kernel_ms_per_step") or 0,1), d.get("host_enqueue_ms_steps"))
    except Exception as e:
        print(f.split("/")[-1], "ERR", open(f).read()[-300:])
PY
