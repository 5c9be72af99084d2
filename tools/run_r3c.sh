mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "strip or shard or peer" > gpurun_out/r3c_tests.log 2>&1
bash tools/multirank_check.sh > gpurun_out/r3c_mr.txt 2>&1
