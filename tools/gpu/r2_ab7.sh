#!/bin/bash
# two-q tiles (TENKIT_STREAM_BQ=1 disables) A/B at cfg3; QR phase trace at 2400x40 / 4000x60 with the
# FP64-tensor-core application for n > 32 (TENKIT_QR_ROWPAR=0: the gathered FFMA one); launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_qr_margins.py -m gpu -q > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/kern_tests.log | head -20
for v in 2 0; do echo "QR ROWPAR=$v"; TENKIT_QR_ROWPAR=$v timeout 120 ./tools/qr_trace 2>&1 | grep -E "per launch|fast path"; done
for C in cfg3; do
  for v in 0 1; do
    TENKIT_STREAM_BQ=$v timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C nobq=$v /"
    TENKIT_STREAM_BQ=$v timeout 900 python bench.py --config $C --steps 8 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C nobq=$v ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 150 -c 4000 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
