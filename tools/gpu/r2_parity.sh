#!/bin/bash
# Full-size oracle parity (cfg3 / cfg4 / cfg5slab) + the new small parity tests + smoke.
mkdir -p gpurun_out
export TENKIT_PARITY_LOG=$PWD/gpurun_out/parity.jsonl
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q -x > gpurun_out/tc_tests.log 2>&1; echo "tc tests rc=$?"; tail -3 gpurun_out/tc_tests.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --durations=0 > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"; tail -15 gpurun_out/fullsize.log
