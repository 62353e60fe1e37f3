#!/bin/bash
# bench lines of the other configs at HEAD + ncu --set full of the cfg5slab passes
mkdir -p gpurun_out
for C in cfg1 cfg2 cfg4 cfg5slab; do
  timeout 1200 python bench.py --config $C > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; echo "$C rc=$?"
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$C.json').read().strip().splitlines()[-1]); print('$C ms/step', d['ms_per_step'], 'value', d['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'], 'e2e', d['e2e']['tucker_ffcp_seconds'], 'floor', d['e2e']['h2d_floor_seconds'])"
done
TENKIT_NO_GRAPH=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ttm_stream_kernel -c 9 -o gpurun_out/prof_cfg5slab_stream \
  python bench.py --config cfg5slab --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full5.log 2>&1; echo "ncu full rc=$?"
