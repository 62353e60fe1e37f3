#!/bin/bash
# round-2 checkpoint: all GPU tests, smoke, default bench (cfg3) + reference arm, ncu launch list
# of one cfg3 step and ncu --set full of its three Y passes (stream kernel)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
rm -f gpurun_out/parity_ckpt.jsonl
TENKIT_PARITY_LOG=gpurun_out/parity_ckpt.jsonl timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; grep -E "^E |passed|failed" gpurun_out/gpu_tests.log | head -8
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_cfg3.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_cfg3.json 2> gpurun_out/bench_ref_cfg3.err; echo "ref rc=$?"; tail -c 1200 gpurun_out/bench_ref_cfg3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 150 -c 4000 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
TENKIT_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttm_stream_kernel -c 9 -o gpurun_out/prof_cfg3_stream \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
