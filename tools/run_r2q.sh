mkdir -p gpurun_out
for DF in 0 1; do
  FSE_DATAFLOW=$DF timeout 600 python tools/bench_configs.py > gpurun_out/r2q_configs_df$DF.txt 2>&1
done
