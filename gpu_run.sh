#!/bin/bash
for v in 0 1; do TENKIT_TC_VARIANT=$v timeout 400 python bench.py --config cfg3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg3.log 2> gpurun_out/bench_cfg3.err; echo "cfg3 v$v rc=$?"; tail -1 gpurun_out/bench_cfg3.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['fit_model'])"; done
