#!/bin/bash
for i in 1 2; do python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
timeout 800 python tools/diag_subspace.py 2>&1 | grep auto
