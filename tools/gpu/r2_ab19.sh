#!/bin/bash
# 12 of 16 rounding adds on the fma pipe (default) vs all 16 (bal16)
mkdir -p gpurun_out
L=$PWD/paper_1412_1885_b200/lib
run() {
  name=$1; lib=$2
  TENKIT_B200_LIB=$lib timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C $name ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'launch ms', d['roofline']['mean_launch_ms'], 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2 3; do
for C in cfg3 cfg4 cfg2 cfg5slab; do
  run bal12 $L/libtenkit_b200.so
  run bal16 $L/libtenkit_b200_bal16.so
done
done
