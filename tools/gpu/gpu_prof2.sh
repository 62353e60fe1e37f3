#!/bin/bash
# Perf + profiles: parity subset, bench, phases, launch list, ncu --set full of the K-major Y pass
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -x -q > gpurun_out/gpu_tests_q.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_q.log
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_perf.log 2> gpurun_out/bench_perf.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_perf.log | cut -c1-300
python tools/phase_bench.py 2>&1 | tail -2
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_perf.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_tc_kernel<32, 1, 1' --launch-skip 2 --launch-count 1 -o gpurun_out/prof_km $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu km rc=$?"
tail -2 gpurun_out/ncu2.log
