#!/bin/bash
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['e2e'])"; tail -3 gpurun_out/bench_q.log | grep -i error
