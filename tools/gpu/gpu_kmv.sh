#!/bin/bash
# K-major Y-pass variant A/B: 256-row tiles, one CTA per SM, 3 accumulator sets (TENKIT_KM_VARIANT=1).
mkdir -p gpurun_out
TENKIT_KM_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_workload.py -q -x > gpurun_out/kmv_t.log 2>&1; rc=$?; echo "tests (variant 1) rc=$rc"; tail -2 gpurun_out/kmv_t.log
for v in 0 1; do
  echo "variant $v"
  TENKIT_KM_VARIANT=$v timeout 300 python tools/phase_bench.py cfg2 2>&1 | tail -2 | head -1
  TENKIT_KM_VARIANT=$v timeout 600 python tools/phase_bench.py cfg4 2>&1 | tail -2 | head -1
done
