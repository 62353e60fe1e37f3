#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_workload.py -q -x -k chunked 2>&1 | tail -2
for c in cfg4 cfg3 cfg1; do timeout 1500 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['fit_model'], d.get('e2e'), d.get('cpu_baseline',{}).get('value'))"; tail -2 gpurun_out/bench_$c.err; done
