# weight-spectrum cache: GPU tests with the cache forced on for every session,
# then the bench with the cache off / on
set -x
mkdir -p gpurun_out
T=${TAG:-s4a}
FSE_WCACHE_ENTRIES=1 timeout 1000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_tests_forced.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests_forced.log
tail -5 gpurun_out/${T}_tests_forced.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
FSE_WCACHE=0 $B > gpurun_out/${T}_bench_wc0.json 2> gpurun_out/${T}_bench_wc0.err
FSE_WCACHE=1 $B > gpurun_out/${T}_bench_wc1.json 2> gpurun_out/${T}_bench_wc1.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/${T}_bench_wc*.json".replace("${T}", __import__("os").environ.get("TAG","s4a")))):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["kernel_ms_per_step"], d.get("weight_spectrum_cache"), d["roofline"]["frac"], d["fp32"]["ms_per_step"])
    except Exception as e:
        print(f, "ERR", e); print(open(f.replace(".json",".err")).read()[-2000:])
PY
