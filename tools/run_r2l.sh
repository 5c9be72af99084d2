mkdir -p gpurun_out
T=${TAG:-r2l}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "128 or config5 or ragged" > gpurun_out/${T}_tests128.log 2>&1
timeout 300 python bench.py --config 5 --block 8 --precision fp64 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c5_b8_fp64.json 2> gpurun_out/${T}_c5_b8_fp64.err
B=8 F=128 WINDOWS=1 python tools/latency_breakdown.py fp64 > gpurun_out/${T}_lat128.jsonl 2>&1 || true
