#!/bin/bash
# A/B: stream kernel with two M tiles per CTA (default) vs one (TENKIT_STREAM_MT=1) vs the r1 kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q -x -k "not fp64_mode" > gpurun_out/stream_tests.log 2>&1; echo "stream tests MT2 rc=$?"; grep -E "^E |passed|failed" gpurun_out/stream_tests.log | head -8
run() {
  name=$1; shift
  env "$@" timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_${C}_$name.log 2> gpurun_out/ab_${C}_$name.err
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
  run r1 TENKIT_STREAM=0
  run mt2 TENKIT_STREAM=1
  run mt1 TENKIT_STREAM_MT=1
  [ $C = cfg5slab ] && run mt2f TENKIT_STREAM_MT=2
done
