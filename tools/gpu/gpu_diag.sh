#!/bin/bash
# Diagnostics: cfg4 leader A/B (phases + launch list), ncu --set full of the cfg2 sketch kernel.
mkdir -p gpurun_out
python tools/phase_bench.py cfg4 > gpurun_out/ph_cfg4.log 2>&1; tail -2 gpurun_out/ph_cfg4.log
TENKIT_NO_KM_LEADER=1 python tools/phase_bench.py cfg4 > gpurun_out/ph_cfg4_nokm.log 2>&1; tail -2 gpurun_out/ph_cfg4_nokm.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/phase_bench.py cfg4 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
TENKIT_NO_KM_LEADER=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_nokm.csv python tools/phase_bench.py cfg4 > gpurun_out/ncu_c4b.log 2>&1; echo "ncu c4b rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sketch_kernel --launch-skip 12 --launch-count 1 -o gpurun_out/prof_sketch python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_sk.log 2>&1; echo "ncu sketch rc=$?"
