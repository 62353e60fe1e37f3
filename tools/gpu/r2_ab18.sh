#!/bin/bash
# hi/lo split spread over both issue pipes (IMAD + LOP3 + immediate-form FFMA, default) vs VIADD + LOP3 + FADD (nobal)
mkdir -p gpurun_out
L=$PWD/paper_1412_1885_b200/lib
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_tc.py -m gpu -q -x > gpurun_out/bal_tests.log 2>&1; echo "stream tests (base) rc=$?"; grep -E "^E |passed|failed" gpurun_out/bal_tests.log | head -5
run() {
  name=$1; lib=$2
  TENKIT_B200_LIB=$lib timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C $name ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'launch ms', d['roofline']['mean_launch_ms'], 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2 3; do
for C in cfg3 cfg4 cfg2 cfg5slab; do
  run bal $L/libtenkit_b200.so
  run nobal $L/libtenkit_b200_nobal.so
done
done
