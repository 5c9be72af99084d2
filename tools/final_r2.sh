# round-2 evidence: GPU tests, smoke, the default bench line (config 4, fp64
# headline with fp32 sub-record, e2e, cpu_baseline), the reference arm, the
# other configs' lines, the ncu launch list of the bench and one --set full
# capture of the fp64 level kernel.  Each ncu command first ran plain.
set -x
mkdir -p gpurun_out
T=${TAG:-r2f}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
for c in 1 2; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_c$c.json 2>&1; done
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3.json 2>&1
python bench.py --config 3 --defaults --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3def.json 2>&1
for B in 2 4 8; do python bench.py --config 5 --block $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_c5_b$B.json 2>&1; done
python tools/cfg5_device.py fp64 2 4 8 > gpurun_out/${T}_cfg5_device.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-second"
$B > gpurun_out/${T}_bench_plain.json 2> gpurun_out/${T}_bench_plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
P="python tools/prof_run.py --frames 16 --precision fp64"
$P > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fse_fast_kernel -s 30 -c 1 -f -o gpurun_out/prof_${T}_f64 $P > gpurun_out/${T}_ncu_f64.log 2>&1
ls -la gpurun_out | tail -30
