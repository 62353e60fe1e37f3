#!/bin/bash
# Stream-kernel variants at cfg3 / cfg2: default, no periodic flush, NH padded to 16; r1 kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # name env...
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
for C in cfg3 cfg2; do
  run r1 TENKIT_STREAM=0
  run stream TENKIT_STREAM=1
  run nochunk TENKIT_STREAM_CHUNK=0
  run nh16 TENKIT_STREAM_NH16=1
  run nochunk_nh16 TENKIT_STREAM_CHUNK=0 TENKIT_STREAM_NH16=1
done
