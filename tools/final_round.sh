#!/bin/bash
# dev: end-of-round measurements: bench lines, reference arm, per-config times, launch list, full captures
bash tools/refresh_bench.sh
bash tools/prof_r1k.sh > gpurun_out/prof_r1k.log 2>&1
