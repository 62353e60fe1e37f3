#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/cfg_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/cfg_tests.log
for c in cfg3 cfg4 cfg1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | cut -c1-260
done
