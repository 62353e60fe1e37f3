#!/bin/bash
# Sketch kernel A/B (cluster vs split + reduce), GPU parity tests, phases, bench.
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests3.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests3.log
python tools/phase_bench.py cfg2 > gpurun_out/ph2.log 2>&1; tail -2 gpurun_out/ph2.log
TENKIT_SKETCH_SPLIT=1 python tools/phase_bench.py cfg2 > gpurun_out/ph2s.log 2>&1; tail -2 gpurun_out/ph2s.log
python tools/phase_bench.py cfg4 > gpurun_out/ph4.log 2>&1; tail -2 gpurun_out/ph4.log
python tools/qr_bench.py > gpurun_out/qr_bench2.log 2>&1; grep gram gpurun_out/qr_bench2.log
python bench.py --steps 30 --no-cpu > gpurun_out/bench_sk.log 2> gpurun_out/bench_sk.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_sk.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_sk.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_sk2.log 2>&1; echo "ncu list rc=$?"
