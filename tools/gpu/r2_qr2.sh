#!/bin/bash
# QR: pivot margin tracked as a fraction (no division / sqrt per Cholesky step), trailing update without
# integer division: parity tests + trace + cfg2 / cfg3 steps
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_qr_margins.py tests/test_gpu_ref_fixtures.py tests/test_gpu_workload.py -m gpu -q > gpurun_out/qr_tests.log 2>&1; echo "tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/qr_tests.log | head
timeout 120 ./tools/qr_trace 2>&1 | grep -E "per launch \(back|fast path|pchol step"
for C in cfg2 cfg3; do
  timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C /"
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
