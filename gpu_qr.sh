#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/qr_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/qr_tests.log
timeout 60 ./tools/qr_trace 2>&1 | grep -E "per launch|fast path|pchol step"
python tools/phase_bench.py 2>&1 | tail -2
