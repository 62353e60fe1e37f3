#!/bin/bash
# A/B in one box: kernel micro-timings and the bench step with the QR variants.
mkdir -p gpurun_out
python tools/kern_bench.py > gpurun_out/kern_bench.log 2>&1; echo "kern rc=$?"; cat gpurun_out/kern_bench.log
TENKIT_QR_ROWPAR=0 python tools/kern_bench.py 2>&1 | grep qr
for v in 1 0 1 0; do
TENKIT_QR_ROWPAR=$v python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('rowpar=$v', d['ms_per_step'], d['clocks']['sm_mhz'])"
done
