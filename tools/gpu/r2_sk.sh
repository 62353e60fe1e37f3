#!/bin/bash
# sketch kernel with one CTA per 32 rows covering all columns (default) vs the 32-column tiles (TENKIT_SKETCH_NARROW=1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workload.py tests/test_gpu_dist.py tests/test_gpu_ref_fixtures.py tests/test_gpu_gram.py -m gpu -q > gpurun_out/sk_tests.log 2>&1; echo "tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/sk_tests.log | head
for C in cfg3 cfg2 cfg4 cfg5slab; do
  for v in 0 1; do
    TENKIT_SKETCH_NARROW=$v timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C narrow=$v /" | cut -c1-230
  done
done
for rep in 1 2; do
for C in cfg3 cfg2; do
  for v in 0 1; do
  TENKIT_SKETCH_NARROW=$v timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C narrow=$v ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
  done
done
done
