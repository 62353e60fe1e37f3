#!/bin/bash
mkdir -p gpurun_out
python tools/qr_bench.py > gpurun_out/qr_bench.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qr_colpiv -s 9 -c 1 -o gpurun_out/prof_qr python tools/qr_bench.py > gpurun_out/ncu_qr.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/qr_bench.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
