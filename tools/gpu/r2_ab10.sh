#!/bin/bash
# y_hi by truncation (TENKIT_STREAM_TRUNC=1) vs round-to-nearest: stream tests, interleaved cfg3 / cfg2 / cfg5slab
# steps, full-size parity (all r~ columns) with the truncating split
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
TENKIT_STREAM_TRUNC=1 timeout 1200 python -m pytest tests/test_gpu_stream.py -m gpu -q > gpurun_out/trunc_tests.log 2>&1; echo "stream tests (trunc) rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/trunc_tests.log | head -20
for rep in 1 2; do
for C in cfg3 cfg2 cfg5slab; do
  for v in 0 1; do
  TENKIT_STREAM_TRUNC=$v timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C trunc=$v ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'launch ms', d['roofline']['mean_launch_ms'], 'clk', d['clocks']['sm_mhz'])"
  done
done
done
rm -f gpurun_out/parity_trunc.jsonl
TENKIT_STREAM_TRUNC=1 TENKIT_PARITY_LOG=gpurun_out/parity_trunc.jsonl timeout 1800 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/fullsize_trunc.log 2>&1; echo "fullsize (trunc) rc=$?"; grep -E "^E |passed|failed" gpurun_out/fullsize_trunc.log | head
