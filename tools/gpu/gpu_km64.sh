#!/bin/bash
# K-major tcgen05 for factors up to 64 columns (NH = 64, one CTA per SM): parity, cfg5slab A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x > gpurun_out/km64_t.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/km64_t.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/km64_fs.log 2>&1; echo "fullsize rc=$?"; tail -1 gpurun_out/km64_fs.log
timeout 600 python tools/phase_bench.py cfg5slab 2>&1 | tail -2 | head -1
TENKIT_KM_LEAD_MAX=64 timeout 600 python tools/phase_bench.py cfg5slab 2>&1 | tail -2
TENKIT_KM_LEAD_MAX=64 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k cfg5 > gpurun_out/km64_fs2.log 2>&1; echo "fullsize km64 lead rc=$?"; grep -E "assert|passed|failed" gpurun_out/km64_fs2.log | tail -3
