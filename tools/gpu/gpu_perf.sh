#!/bin/bash
# Perf iteration: quick parity subset, bench, launch list, QR phase trace.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -x -q > gpurun_out/gpu_tests_q.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/gpu_tests_q.log
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_perf.log 2> gpurun_out/bench_perf.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_perf.log | cut -c1-300
python tools/phase_bench.py > gpurun_out/phases.log 2>&1; echo "phases rc=$?"; cat gpurun_out/phases.log | tail -3
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_perf.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "ncu rc=$?"
timeout 60 ./tools/qr_trace > gpurun_out/qr_trace.log 2>&1; echo "qr_trace rc=$?"; cat gpurun_out/qr_trace.log | head -20
