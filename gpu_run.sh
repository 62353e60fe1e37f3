#!/bin/bash
python tools/ffcp_bench.py 200 > gpurun_out/ffcp.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ffcp_launches.csv python tools/ffcp_bench.py 3 > /dev/null 2>&1
cat gpurun_out/ffcp.log
