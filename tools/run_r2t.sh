mkdir -p gpurun_out
T=r2t
for v in main gen128; do
  lib=""; [ $v = gen128 ] && lib=paper_2207_00233_b200/variants/libfse_b200_gen128.so
  FSE_LIB=$lib timeout 400 python bench.py --config 5 --block 8 --precision fp64 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c5b8_$v.json 2>&1
done
python tools/setup_share.py 16 fp64 > gpurun_out/${T}_setup_share.txt 2>&1 || true
