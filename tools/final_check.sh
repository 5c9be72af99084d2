#!/bin/bash
# dev: final round checks: GPU tests, smoke, bench lines, multi-rank functional run
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
python bench.py > gpurun_out/final/bench_full.json 2> gpurun_out/final/bench_full.err
for b in 2 4 8; do python bench.py --config 5 --block $b > gpurun_out/final/bench_c5_b$b.json 2>&1; done
bash tools/multirank_check.sh > gpurun_out/final/mr_summary.txt 2>&1; cp gpurun_out/mr_*.json gpurun_out/final/ 2>/dev/null
