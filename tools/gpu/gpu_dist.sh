#!/bin/bash
# Multi-rank bench code paths on one GPU (ranks share the device over gloo: a code-path check,
# not a scaling number): 2-rank slabs and the 8-rank 2x2x2 block grid, small config first.
mkdir -p gpurun_out
for cfg in cfg1 cfg2; do for n in 2 8; do
TENKIT_BENCH_GLOO=1 timeout 300 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n \
  bench.py --gpus $n --steps 3 --warmup 3 --no-e2e --config $cfg > gpurun_out/bench_${cfg}_g$n.log 2> gpurun_out/bench_${cfg}_g$n.err; echo "$cfg g$n rc=$?"
tail -1 gpurun_out/bench_${cfg}_g$n.log | cut -c1-700
grep "^\[rank" gpurun_out/bench_${cfg}_g$n.err | tail -4
done; done
