#!/bin/bash
# Shared-pass step groups: full GPU tests, bench (grouped and one-pass-per-step A/B), ncu launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/gpu_tests.log
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_grp.log 2> gpurun_out/bench_grp.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_grp.log | cut -c1-420
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --one-pass-per-step > gpurun_out/bench_ungrp.log 2>&1; echo "bench ungrouped rc=$?"
tail -1 gpurun_out/bench_ungrp.log | cut -c1-420
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_grp.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "ncu rc=$?"
TENKIT_BENCH_GLOO=1 timeout 400 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_cfg2_g2.log 2> gpurun_out/bench_cfg2_g2.err; echo "g2 rc=$?"
tail -1 gpurun_out/bench_cfg2_g2.log | cut -c1-600
