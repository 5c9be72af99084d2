#!/bin/bash
# dev: device-resident bench step vs the first planned chunk (plan_and_run)
mkdir -p gpurun_out
for c in 0 16 32 64; do for rep in 1 2; do FSE_FIRST_CHUNK=$c python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('first_chunk $c', round(d['ms_per_step'],2), round(d['kernel_ms_per_step'],2), round(d['fp64']['ms_per_step'],2), round(d['fp64']['kernel_ms_per_step'],2))"; done; done > gpurun_out/chunk_sweep.txt 2>&1
