#!/bin/bash
# A/B kernel ms of the product library against variants/libfse_b200_<tag>.so
# usage (on the GPU box): tools/ab.sh tag [tag2 ...]   extra bench args via AB_ARGS
for rep in 1 2; do
  for v in main "$@"; do
    if [ "$v" = main ]; then lib=""; else lib="paper_2207_00233_b200/variants/libfse_b200_$v.so"; fi
    FSE_LIB=$lib python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $AB_ARGS > /tmp/ab.log 2>&1
    python -c "
import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1])
s=d.get('fp64') or d.get('fp32') or {}
print('$v', d['dtype'], round(d['kernel_ms_per_step'],2), round(d['roofline']['frac'],4), 'other', round(s.get('kernel_ms_per_step',0),2))" || tail -3 /tmp/ab.log
  done
done
