#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_tc_kernel<\(int\)32, \(int\)1, \(bool\)1' --launch-skip 2 --launch-count 1 -o gpurun_out/prof_km $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu km rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_tc_kernel<\(int\)32, \(int\)2, \(bool\)0' --launch-skip 2 --launch-count 1 -o gpurun_out/prof_mm $CMD > gpurun_out/ncu3.log 2>&1; echo "ncu mm rc=$?"
ls -la gpurun_out/*.ncu-rep
