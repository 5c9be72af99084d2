#!/bin/bash
# dev: GPU tests + per-config device times + one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest.log
python tools/bench_configs.py > gpurun_out/g_cfg.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench.json 2>&1
