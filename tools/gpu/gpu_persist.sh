#!/bin/bash
# Persistent tcgen05 TTM (tile loop) A/B: parity first (bounded), then phases and bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x > gpurun_out/gpu_tests6.log 2>&1; rc=$?; echo "tc/parity tests rc=$rc"; tail -3 gpurun_out/gpu_tests6.log
if [ $rc -ne 0 ]; then exit 1; fi
for v in 1 0; do
  echo "persist=$v"
  TENKIT_TC_PERSIST=$v timeout 300 python tools/phase_bench.py cfg2 2>&1 | tail -2 | head -1
  TENKIT_TC_PERSIST=$v timeout 600 python tools/phase_bench.py cfg4 2>&1 | tail -2 | head -1
  TENKIT_TC_PERSIST=$v timeout 600 python tools/phase_bench.py cfg3 2>&1 | tail -2 | head -1
done
timeout 600 python bench.py --steps 30 --no-cpu > gpurun_out/bench_p.log 2> gpurun_out/bench_p.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'], d['clocks'])"
