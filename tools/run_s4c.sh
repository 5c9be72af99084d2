# weight-spectrum cache, second pass: tests with every window cached, bench off / on, fp32 open timing
set -x
mkdir -p gpurun_out
T=${TAG:-s4c}
FSE_WCACHE_ENTRIES=1 FSE_WCACHE_MIN=1 timeout 1000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_tests_forced.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests_forced.log
tail -5 gpurun_out/${T}_tests_forced.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
FSE_WCACHE=0 $B > gpurun_out/${T}_bench_wc0.json 2> gpurun_out/${T}_bench_wc0.err
FSE_WCACHE=1 $B > gpurun_out/${T}_bench_wc1.json 2> gpurun_out/${T}_bench_wc1.err
FSE_WCACHE=1 FSE_WCACHE_PLANES=16384 $B --no-second > gpurun_out/${T}_bench_wc1_16k.json 2> gpurun_out/${T}_bench_wc1_16k.err
FSE_OPEN_TIMING=1 FSE_WCACHE=1 $B --precision fp32 --no-second > gpurun_out/${T}_bench_f32_wc1.json 2> gpurun_out/${T}_bench_f32_wc1.err
FSE_OPEN_TIMING=1 FSE_WCACHE=0 $B --precision fp32 --no-second > gpurun_out/${T}_bench_f32_wc0.json 2> gpurun_out/${T}_bench_f32_wc0.err
tail -8 gpurun_out/${T}_bench_f32_wc1.err gpurun_out/${T}_bench_f32_wc0.err
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s4c")
for f in sorted(glob.glob(f"gpurun_out/{T}_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        o=d.get("fp32") or {}
        print(f, d["dtype"], round(d["ms_per_step"],1), round(d["kernel_ms_per_step"],1), d.get("weight_spectrum_cache"), round(d["roofline"]["frac"],4), "enq", round(d["host_enqueue_ms_per_step"],1), "other", o.get("ms_per_step"), o.get("kernel_ms_per_step"))
    except Exception as e:
        print(f, "ERR", e); print(open(f.replace(".json",".err")).read()[-2000:])
PY
