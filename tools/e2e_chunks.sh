#!/bin/bash
# dev: e2e wall time per conceal_batch call for chunk schedules (FSE_CHUNKS)
mkdir -p gpurun_out
for c in "" "0.0625,0.875,0.0625" "0.03125,0.90625,0.0625" "0.0625,0.90625,0.03125" "0.09375,0.84375,0.0625"; do
  echo "== FSE_CHUNKS=$c" >> gpurun_out/e2e_chunks3.txt
  CALLS=12 FSE_CHUNKS=$c python tools/e2e_calls.py >> gpurun_out/e2e_chunks3.txt 2>&1
done
