#!/bin/bash
for v in 0 1; do TENKIT_TC_VARIANT=$v python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_q.log 2>&1; echo "variant $v: $(tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'])")"; done
timeout 300 python tools/diag_ttm_err.py
timeout 800 python tools/diag_subspace.py 2>&1 | grep auto
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
