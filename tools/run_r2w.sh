mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2w_tests.log 2>&1
for rep in 1 2; do
for v in main gen12; do
  lib=""; [ $v != main ] && lib=paper_2207_00233_b200/variants/libfse_b200_$v.so
  FSE_LIB=$lib timeout 300 python bench.py --config 3 --defaults --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-second > /tmp/d.json 2>&1
  python -c "
import json; d=json.loads(open('/tmp/d.json').read().strip().splitlines()[-1]); print('$v', round(d['kernel_ms_per_step'],3), round(d['ms_per_step'],3))" >> gpurun_out/r2w_ab.txt
done
done
