#!/bin/bash
# ncu launch lists of one step of cfg4 / cfg2 / cfg5slab
mkdir -p gpurun_out
for C in cfg4 cfg2 cfg5slab; do
  skip=150; [ $C = cfg4 ] && skip=60
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip $skip -c 4000 --csv --log-file gpurun_out/launches_$C.csv \
    python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches_$C.log 2>&1; echo "$C launch list rc=$?"
done
