mkdir -p gpurun_out
for v in main track; do
  if [ $v = main ]; then lib=""; else lib=paper_2207_00233_b200/variants/libfse_b200_$v.so; fi
  echo "== $v" >> gpurun_out/cfgab.txt
  FSE_LIB=$lib python tools/bench_configs.py 2 3 5 >> gpurun_out/cfgab.txt 2>&1
done
