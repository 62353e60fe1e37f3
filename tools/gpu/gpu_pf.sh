#!/bin/bash
# L2 prefetch distance A/B for the persistent tcgen05 Y passes.
mkdir -p gpurun_out
for v in 0 8 16 32; do
  echo "l2pf=$v"
  TENKIT_TC_L2PF=$v timeout 300 python tools/phase_bench.py cfg2 2>&1 | tail -2 | head -1
  TENKIT_TC_L2PF=$v timeout 600 python tools/phase_bench.py cfg4 2>&1 | tail -2 | head -1
done
TENKIT_TC_L2PF=16 timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/gpu_tests7.log 2>&1; echo "tc tests (pf16) rc=$?"; tail -1 gpurun_out/gpu_tests7.log
