mkdir -p gpurun_out
for v in 0 12 22; do
  for c in 1 2; do
    FSE_F64L=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2n_c${c}_f64l$v.json 2>&1
  done
done
