#!/bin/bash
# Sketch split-K target A/B (CTAs per grid), full GPU tests.
mkdir -p gpurun_out
for t in 592 296 1184; do
  echo "target $t"; TENKIT_SKETCH_CTAS=$t python tools/phase_bench.py cfg2 2>&1 | tail -2 | head -1
  TENKIT_SKETCH_CTAS=$t python tools/phase_bench.py cfg4 2>&1 | tail -2 | head -1
done
timeout 1300 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests5.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests5.log
