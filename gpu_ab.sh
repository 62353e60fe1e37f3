#!/bin/bash
for v in 1 0 1 0; do echo "CARVEOUT=$v"; TENKIT_CARVEOUT=$v python tools/phase_bench.py 2>&1 | grep phases | tail -1; done
for v in 1 0 1 0; do TENKIT_CARVEOUT=$v python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('carveout=$v', d['ms_per_step'], d['clocks']['sm_mhz'])"; done
