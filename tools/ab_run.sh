#!/bin/bash
# dev: GPU tests against variant libraries, then A/B kernel timings (tools/ab.sh)
# usage: tools/ab_run.sh tag [tag2 ...]
mkdir -p gpurun_out
for v in "$@"; do
  FSE_LIB=paper_2207_00233_b200/variants/libfse_b200_$v.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest_$v.log 2>&1
  echo "$v pytest rc=$?" >> gpurun_out/ab_summary.txt
  tail -2 gpurun_out/ab_pytest_$v.log >> gpurun_out/ab_summary.txt
done
bash tools/ab.sh "$@" >> gpurun_out/ab_summary.txt 2>&1
