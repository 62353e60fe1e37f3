#!/bin/bash
timeout 300 python tools/qr_bench.py
TENKIT_QR_NO_FAST=1 timeout 300 python tools/qr_bench.py
timeout 900 python -m pytest tests -m gpu -q -x -k "qr or basis or golden or parity or tc or workload" 2>&1 | tail -3
python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'])"
timeout 800 python tools/diag_subspace.py 2>&1 | grep auto
