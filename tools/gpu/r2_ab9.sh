#!/bin/bash
# trimmed converter loop (register-held barrier addresses, immediate LDS offsets): tests + cfg3/cfg2/cfg5slab steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_tc.py -m gpu -q > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/kern_tests.log | head -20
for C in cfg3 cfg2 cfg5slab cfg3; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'launch ms', d['roofline']['mean_launch_ms'], 'clk', d['clocks']['sm_mhz'])"
  timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C /"
done
