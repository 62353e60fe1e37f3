#!/bin/bash
# A/B of the Y-pass kernels on every bench config: TENKIT_STREAM=0 (round-1 kernel) vs the stream kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q -x -k "not fp64_mode" > gpurun_out/stream_tests.log 2>&1; echo "stream tests rc=$?"; grep -E "^E |passed|failed" gpurun_out/stream_tests.log | head -8
for c in cfg3 cfg2 cfg5slab cfg4; do
  for v in 0 1; do
    TENKIT_STREAM=$v timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_$v.log 2> gpurun_out/bench_${c}_$v.err
    python - $c $v <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/bench_{c}_{v}.log").read().strip().splitlines()[-1])
    print(c, "stream" if v == "1" else "r1", "ms/step", d["ms_per_step"], "kernel frac", d["roofline"]["frac"], "mean launch ms", d["roofline"]["mean_launch_ms"], "clk", d["clocks"]["sm_mhz"], "fit", d["fit_model"])
except Exception as e:
    print(c, v, "failed", e)
PY
  done
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_stream_kernel' --launch-count 1 -o gpurun_out/r2_cfg3_ts python tools/one_decomp.py cfg3 > gpurun_out/ncu_stream.log 2>&1; echo "ncu rc=$?"
