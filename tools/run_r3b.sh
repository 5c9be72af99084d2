mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3b_tests.log 2>&1
for PDL in 1 0; do
  for c in 1 2; do FSE_PDL=$PDL timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r3b_c${c}_pdl$PDL.json 2>&1; done
  FSE_PDL=$PDL python tools/cfg5_device.py fp64 2 4 8 > gpurun_out/r3b_cfg5_pdl$PDL.txt 2>&1
  FSE_PDL=$PDL timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-second > gpurun_out/r3b_c4_pdl$PDL.json 2>&1
  FSE_PDL=$PDL timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/r3b_c3_pdl$PDL.json 2>&1
done
