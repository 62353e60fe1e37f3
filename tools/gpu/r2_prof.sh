#!/bin/bash
# ncu --set full of one Y pass: the r1 kernel vs the stream kernel (cfg2 and cfg3), with source
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NCU="ncu --set full --clock-control none --import-source on -c 1"
for C in cfg2 cfg3; do
  TENKIT_STREAM=0 timeout 600 $NCU -k regex:ttm_tc_kernel -o gpurun_out/prof_${C}_r1 python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_${C}_r1.log 2>&1; echo "$C r1 rc=$?"
  timeout 600 $NCU -k regex:ttm_stream_kernel -o gpurun_out/prof_${C}_st python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_${C}_st.log 2>&1; echo "$C st rc=$?"
done
