#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -5
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench rc=$?"
cat gpurun_out/bench_full.log; tail -3 gpurun_out/bench_full.err
