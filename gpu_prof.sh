#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:ttm_tc_kernel -s 6 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc=$?"
tail -1 gpurun_out/plain.log | cut -c1-300
