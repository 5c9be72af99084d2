set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j_bench_plain.json 2> gpurun_out/j_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1k.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j_ncu_launch.log 2>&1
python tools/prof_run.py --frames 16 > /dev/null 2>&1 || exit 2
ncu --set full --clock-control none --import-source on -k regex:fse_fast_kernel -s 30 -c 1 -f -o gpurun_out/prof_r1k_f32 python tools/prof_run.py --frames 16 > gpurun_out/j_ncu_f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fse_fast_kernel -s 30 -c 1 -f -o gpurun_out/prof_r1k_f64 python tools/prof_run.py --frames 16 --precision fp64 > gpurun_out/j_ncu_f64.log 2>&1
ls -la gpurun_out
