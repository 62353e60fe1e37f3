#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ffcp_exp.py > gpurun_out/ffcp_exp.log 2>&1; echo "exp rc=$?"; tail -4 gpurun_out/ffcp_exp.log
timeout 300 python tools/ffcp_bench.py 200 > gpurun_out/ffcp.log 2>&1; echo "ffcp rc=$?"
cat gpurun_out/ffcp.log
timeout 900 python -m pytest tests -m gpu -q -x -k "ffcp or golden or cpp or workload" 2>&1 | tail -5
