#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['e2e'], d['cpu_baseline']['value'])"
