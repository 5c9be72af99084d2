# round 2 evidence run (one B200): GPU tests, per-level latency calibration,
# per-config device times, the bench launch list under ncu, and ncu --set full
# captures of the fp64 headline kernel (wide config-4 level) and of the
# any-size kernel on the reference-default drop-in call (config 3 frame).
# Every ncu command first ran plain (exit 0) in this same script.
set -x
mkdir -p gpurun_out
T=${TAG:-r2j}
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
python tools/window_latency.py > gpurun_out/${T}_latency.jsonl 2>&1
python tools/bench_configs.py > gpurun_out/${T}_configs.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-second"
$B > gpurun_out/${T}_bench_plain.json 2> gpurun_out/${T}_bench_plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
P="python tools/prof_run.py --frames 16 --precision fp64"
$P > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fse_fast_kernel -s 30 -c 1 -f -o gpurun_out/prof_${T}_f64 $P > gpurun_out/${T}_ncu_f64.log 2>&1
D="python bench.py --config 3 --defaults --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-second"
$D > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fse_gen_kernel -s 2 -c 1 -f -o gpurun_out/prof_${T}_gen $D > gpurun_out/${T}_ncu_gen.log 2>&1
ls -la gpurun_out | tail -20
