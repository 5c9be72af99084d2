# round 2 profiling: per-config device times, then ncu --set full of an fp64
# wide config-4 level and a narrow config-1 level (each command first run plain)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2c}
python tools/bench_configs.py > gpurun_out/${TAG}_configs.txt 2>&1
python tools/prof_run.py --frames 16 --precision fp64 > /dev/null 2>&1 || exit 2
ncu --set full --clock-control none --import-source on -k regex:fse_fast_kernel -s 30 -c 1 -f -o gpurun_out/prof_${TAG}_f64 python tools/prof_run.py --frames 16 --precision fp64 > gpurun_out/${TAG}_ncu_f64.log 2>&1
python tools/prof_run.py --config 1 --frames 1 --precision fp64 > /dev/null 2>&1 || exit 3
ncu --set full --clock-control none --import-source on -k regex:fse_fast_kernel -s 5 -c 1 -f -o gpurun_out/prof_${TAG}_c1 python tools/prof_run.py --config 1 --frames 1 --precision fp64 > gpurun_out/${TAG}_ncu_c1.log 2>&1
