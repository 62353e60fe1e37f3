#!/bin/bash
mkdir -p gpurun_out
TENKIT_BENCH_GLOO=1 timeout 900 torchrun --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29538 \
  bench.py --gpus 8 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_cfg2_g8.log 2> gpurun_out/bench_cfg2_g8.err; echo "g8 rc=$?"
tail -1 gpurun_out/bench_cfg2_g8.log | cut -c1-900
grep "^\[rank" gpurun_out/bench_cfg2_g8.err | tail -3
