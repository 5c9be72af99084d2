#!/bin/bash
# dev: refresh the committed bench lines (profiles/bench_r1) on one GPU
mkdir -p gpurun_out/bench
python bench.py > gpurun_out/bench/bench_full.json 2> gpurun_out/bench/bench_full.err
python bench.py --impl reference > gpurun_out/bench/ref_full.json 2> gpurun_out/bench/ref_full.err
python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench/bench_c1.json 2>&1
python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench/bench_c2.json 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench/bench_c3.json 2>&1
for b in 2 4 8; do python bench.py --config 5 --block $b > gpurun_out/bench/bench_c5_b$b.json 2>&1; done
python tools/bench_configs.py > gpurun_out/bench/configs.txt 2>&1
