mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2y_tests.log 2>&1
for c in 1 2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2y_c$c.json 2>&1; done
