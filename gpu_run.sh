#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/qr_bench.py > gpurun_out/qr.log 2>&1; cat gpurun_out/qr.log
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['e2e'])"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
