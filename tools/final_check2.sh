#!/bin/bash
# dev: last checks of the round (GPU tests, smoke, default bench, reference arm)
mkdir -p gpurun_out/final2
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
python bench.py > gpurun_out/final2/bench_full.json 2> gpurun_out/final2/bench_full.err; echo "bench rc=$?" >> gpurun_out/final2/smoke.log
python bench.py --impl reference > gpurun_out/final2/ref_full.json 2> gpurun_out/final2/ref_full.err; echo "ref rc=$?" >> gpurun_out/final2/smoke.log
