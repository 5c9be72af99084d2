# plan thread count inside the bench steps (config 5 B=2 fp32, config 3 fp64)
mkdir -p gpurun_out
for T in 1 8 12 16; do
  FSE_PLAN_THREADS=$T timeout 300 python bench.py --config 5 --block 2 --precision fp32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/r2k_c5b2_t$T.json 2>&1
  FSE_PLAN_THREADS=$T timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/r2k_c3_t$T.json 2>&1
done
