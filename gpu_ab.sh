#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_workload.py tests/test_golden.py -x -q 2>&1 | tail -2
for v in 1 2; do python tools/phase_bench.py 2>&1 | grep phases | tail -1; done
python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | cut -c1-220
