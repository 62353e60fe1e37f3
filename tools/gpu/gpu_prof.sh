#!/bin/bash
# Bench + profiles: plain bench run, then (same command exited 0) the ncu launch list and one
# ncu --set full capture of the Y-streaming tcgen05 kernel.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log | cut -c1-300
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
  echo "ncu1 rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:ttm_tc_kernel -s 6 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu2.log 2>&1
  echo "ncu2 rc=$?"
fi
