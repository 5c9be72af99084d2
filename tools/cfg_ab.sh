#!/bin/bash
# dev: per-config device times of the product library and variant libraries
# usage: tools/cfg_ab.sh "configs" tag...
mkdir -p gpurun_out
cfgs=$1; shift
for v in main "$@"; do
  if [ $v = main ]; then lib=""; else lib=paper_2207_00233_b200/variants/libfse_b200_$v.so; fi
  echo "== $v" >> gpurun_out/cfgab.txt
  FSE_LIB=$lib python tools/bench_configs.py $cfgs >> gpurun_out/cfgab.txt 2>&1
done
