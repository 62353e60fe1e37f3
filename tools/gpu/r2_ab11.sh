#!/bin/bash
# compile-time sensitivity of the stream kernel (variant libraries from tools/build_variant.sh, selected
# with TENKIT_B200_LIB): A-buffer ring depth, stage ring depth, chunk length, one accumulator buffer
mkdir -p gpurun_out
L=$PWD/paper_1412_1885_b200/lib
run() {
  name=$1; lib=$2
  TENKIT_B200_LIB=$lib timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C $name ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'launch ms', d['roofline']['mean_launch_ms'], 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
for C in cfg3 cfg2; do
  run base $L/libtenkit_b200.so
  for v in na2 st6 ch32 nd1; do run $v $L/libtenkit_b200_$v.so; done
done
done
python tools/ffcp_bench.py 200 40 2400 30 2>&1 | grep -E "kind 0|kind 2"
