# round-2 bench lines of the non-headline configs (planner now band-parallel)
mkdir -p gpurun_out
T=${TAG:-r2j}
for B in 2 4 8; do
  for PR in fp32 fp64; do
    timeout 300 python bench.py --config 5 --block $B --precision $PR --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c5_b${B}_${PR}.json 2> gpurun_out/${T}_c5_b${B}_${PR}.err
  done
done
timeout 300 python bench.py --config 3 --defaults --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3_defaults.json 2> gpurun_out/${T}_c3_defaults.err
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c1.json 2> gpurun_out/${T}_c1.err
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
