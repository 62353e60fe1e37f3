#!/bin/bash
for gr in 0 1 0 1; do TENKIT_NO_GRAPH=$gr timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_q.log 2> gpurun_out/bench_q.err; echo "no_graph=$gr $(tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])")"; done
