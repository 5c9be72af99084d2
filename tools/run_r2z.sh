mkdir -p gpurun_out
for v in main d32w3 d32w3m6; do
  lib=""; [ $v != main ] && lib=paper_2207_00233_b200/variants/libfse_b200_$v.so
  TAGV=$v FSE_LIB=$lib python tools/cfg5_device.py fp64 2 >> gpurun_out/r2z_ab.txt 2>&1
done
for v in main d128lg3; do
  lib=""; [ $v != main ] && lib=paper_2207_00233_b200/variants/libfse_b200_$v.so
  TAGV=$v FSE_LIB=$lib python tools/cfg5_device.py fp64 8 >> gpurun_out/r2z_ab.txt 2>&1
done
