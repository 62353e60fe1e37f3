#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_workload.py -x -q > gpurun_out/qr_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/qr_tests.log
timeout 60 ./tools/qr_trace 2>&1 | grep -E "per launch|fast path|pchol step"
python tools/phase_bench.py 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | cut -c1-250
