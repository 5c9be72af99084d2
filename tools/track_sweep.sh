#!/bin/bash
# dev: config 4 kernel time vs the tracked/lazy threshold (FSE_TRACK_BELOW)
mkdir -p gpurun_out
for t in 0 1184 2368 4736 9472 100000000; do FSE_TRACK_BELOW=$t python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('below $t', round(d['kernel_ms_per_step'],2), round(d['fp64']['kernel_ms_per_step'],2))"; done > gpurun_out/track_sweep.txt 2>&1
