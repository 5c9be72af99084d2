mkdir -p gpurun_out
for v in main solooff solo2 solo8 solo16; do
  lib=""; [ $v != main ] && lib=paper_2207_00233_b200/variants/libfse_b200_$v.so
  echo "== $v" >> gpurun_out/r3d_plan.txt
  FSE_LIB=$lib python tools/plan_threads_time.py 12 16 >> gpurun_out/r3d_plan.txt 2>&1
done
