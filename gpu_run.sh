#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg4.log 2>&1; tail -1 gpurun_out/bench_cfg4.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['fit_model'], d['e2e']['tucker_ffcp_seconds'])"
