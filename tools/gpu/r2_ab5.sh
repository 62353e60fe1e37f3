#!/bin/bash
# blocked tall-sketch QR tests; stream-kernel converter prefetch A/B (TENKIT_STREAM_PF) on every config
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_qr_margins.py tests/test_gpu_stream.py tests/test_gpu_tc.py -m gpu -q > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/kern_tests.log | head -20
run() {
  name=$1; shift
  env "$@" timeout 900 python bench.py --config $C --steps 8 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_${C}_$name.log 2> gpurun_out/ab_${C}_$name.err
  python - $C $name <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{c}_{v}.log").read().strip().splitlines()[-1])
    print(c, v, "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"], "launch ms", d["roofline"]["mean_launch_ms"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(c, v, "failed", e)
PY
}
for C in cfg3 cfg2 cfg4 cfg5slab; do
  run pf1 TENKIT_STREAM_PF=1
  run pf0 TENKIT_STREAM_PF=0
  TENKIT_STREAM_PF=1 timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C pf1 /"
  TENKIT_STREAM_PF=0 timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C pf0 /"
done
