#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_workload.py -x -q > gpurun_out/km_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/km_tests.log
python tools/phase_bench.py 2>&1 | grep phases | tail -1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | cut -c1-200
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_km.csv $CMD > /dev/null 2>&1; echo "ncu rc=$?"
