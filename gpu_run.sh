#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain20.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/plain20.log | cut -c1-200; grep -o '"roofline": {[^}]*}' gpurun_out/plain20.log; grep -o '"fit_model": [0-9.]*' gpurun_out/plain20.log
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -x -q 2>&1 | tail -2
