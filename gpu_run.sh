#!/bin/bash
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  ncu --set full --clock-control none -k regex:sketch_kernel -s 20 -c 1 -o gpurun_out/prof_sketch $CMD > gpurun_out/ncu3.log 2>&1
  echo "ncu rc=$?"
fi
