#!/bin/bash
# Round-1 final checkpoint (after the persistent TTM): smoke, all GPU tests, benches, phases, ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_cfg2.log | cut -c1-200
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for c in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
python tools/phase_bench.py > gpurun_out/phases.log 2>&1; tail -2 gpurun_out/phases.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_tc_kernel<\(int\)32, \(int\)2, \(bool\)0' --launch-skip 2 --launch-count 1 -o gpurun_out/prof_mm $CMD > gpurun_out/ncu3.log 2>&1; echo "ncu mm rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_tc_kernel<\(int\)32, \(int\)1, \(bool\)1' --launch-skip 2 --launch-count 1 -o gpurun_out/prof_km $CMD > gpurun_out/ncu5.log 2>&1; echo "ncu km rc=$?"
