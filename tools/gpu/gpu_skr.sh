#!/bin/bash
# Sketch with the last-CTA reduction: parity tests, phases A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_dist.py -q -x > gpurun_out/gpu_tests8.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/gpu_tests8.log
for v in 0 1; do
  echo "split reduce=$v"
  TENKIT_SKETCH_REDUCE=$v timeout 300 python tools/phase_bench.py cfg2 2>&1 | tail -2 | head -1
  TENKIT_SKETCH_REDUCE=$v timeout 600 python tools/phase_bench.py cfg4 2>&1 | tail -2 | head -1
done
