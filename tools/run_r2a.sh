set -x
mkdir -p gpurun_out
T=r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
