#!/bin/bash
# dev: e2e wall time per conceal_batch call
mkdir -p gpurun_out
CALLS=24 FSE_E2E_TRACE=1 python tools/e2e_calls.py > gpurun_out/e2e_pool.txt 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-second > gpurun_out/e2e_pool_bench.json 2>&1
