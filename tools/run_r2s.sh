mkdir -p gpurun_out
T=r2s
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
bash tools/multirank_check.sh > gpurun_out/${T}_mr.txt 2>&1
for B in 2 4 8; do
  for PR in fp64 fp32; do
    timeout 300 python bench.py --config 5 --block $B --precision $PR --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c5_b${B}_${PR}.json 2> gpurun_out/${T}_c5_b${B}_${PR}.err
  done
done
