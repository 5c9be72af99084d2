#!/bin/bash
# dev: e2e wall time per conceal_batch call for chunk schedules (FSE_CHUNKS)
mkdir -p gpurun_out
for c in "" "0.125,0.8125,0.0625" "0.125,0.84375,0.03125" "0.09375,0.84375,0.0625" "0.125,0.75,0.125"; do
  echo "== FSE_CHUNKS=$c" >> gpurun_out/e2e_chunks2.txt
  CALLS=12 FSE_CHUNKS=$c python tools/e2e_calls.py >> gpurun_out/e2e_chunks2.txt 2>&1
done
