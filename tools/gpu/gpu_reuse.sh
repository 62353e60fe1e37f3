#!/bin/bash
# First-contraction reuse across a group's steps (N = 4): parity tests and cfg4 phases A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_gram.py -q -x > gpurun_out/gpu_tests4.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests4.log
python tools/phase_bench.py cfg4 > gpurun_out/ph4r.log 2>&1; tail -2 gpurun_out/ph4r.log
TENKIT_NO_REUSE=1 python tools/phase_bench.py cfg4 > gpurun_out/ph4n.log 2>&1; tail -2 gpurun_out/ph4n.log
timeout 900 python bench.py --config cfg4 --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_cfg4r.log 2> gpurun_out/bench_cfg4r.err; echo "cfg4 rc=$?"; tail -1 gpurun_out/bench_cfg4r.log | cut -c1-300
