#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_workload.py -x -q -s > gpurun_out/pytest_workload.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_workload.log
tail -30 gpurun_out/pytest_workload.log
