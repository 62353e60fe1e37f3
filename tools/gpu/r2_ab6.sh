#!/bin/bash
# tall QR + host-landing tests; packed-split (TENKIT_STREAM_V2) A/B; e2e with / without slab landing;
# launch list + ncu --set full of the cfg3 Y passes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_qr_margins.py tests/test_gpu_stream.py -m gpu -q > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/kern_tests.log | head -20
TENKIT_STREAM_V2=1 timeout 1200 python -m pytest tests/test_gpu_stream.py -m gpu -q > gpurun_out/v2_tests.log 2>&1; echo "V2 stream tests rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/v2_tests.log | head -20
run() {
  name=$1; shift
  env "$@" timeout 900 python bench.py --config $C --steps 8 --warmup 3 $E2E --no-cpu > gpurun_out/ab_${C}_$name.log 2> gpurun_out/ab_${C}_$name.err
  python - $C $name <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{c}_{v}.log").read().strip().splitlines()[-1])
    print(c, v, "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"], "launch ms", d["roofline"]["mean_launch_ms"], "clk", d["clocks"]["sm_mhz"],
          "e2e", d.get("e2e", {}).get("tucker_ffcp_seconds"), "floor", d.get("e2e", {}).get("h2d_floor_seconds"))
except Exception as e:
    print(c, v, "failed", e)
PY
}
E2E=--no-e2e
for C in cfg3 cfg2 cfg4 cfg5slab; do
  run v2 TENKIT_STREAM_V2=1
  run v1 TENKIT_STREAM_V2=0
  TENKIT_STREAM_V2=1 timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C v2 /"
done
E2E=
for C in cfg3 cfg2; do
  run land8 TENKIT_LAND_SLABS=8
  run land1 TENKIT_LAND_SLABS=1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tkb" -c 4000 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
TENKIT_NO_GRAPH=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ttm_stream_kernel -c 9 -o gpurun_out/prof_cfg3_stream9 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
