#!/bin/bash
# dev: 2-rank functional check of bench.py on ONE GPU (gloo reductions; the
# ranks share the GPU, so the numbers are not scaling results)
mkdir -p gpurun_out
export FSE_BENCH_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/mr_c4.json 2> gpurun_out/mr_c4.err; echo "c4 rc=$?"
timeout 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --config 5 --block 4 --no-cpu-baseline > gpurun_out/mr_c5.json 2> gpurun_out/mr_c5.err; echo "c5 rc=$?"
timeout 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --config 5 --block 4 --halo collective --no-cpu-baseline > gpurun_out/mr_c5c.json 2> gpurun_out/mr_c5c.err; echo "c5 collective rc=$?"
timeout 900 $R bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"
